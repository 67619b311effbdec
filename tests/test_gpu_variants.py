"""Solver-plumbing switches that must not change a single bit (DESIGN.md
§6b): host-driven GMRES columns instead of CUDA-graph WHILE nodes, the fused
cooperative coarse V-cycle, the un-fused first fine Jacobi sweep, and the
line search without the watched-row pre-check, the restriction in
launches of its own, and line-search trials evaluated without the Jacobian
blocks (the accepted trial's element pass is then repeated at the next Newton
point).  Each
variant runs in its own process (the switches are read when the library
loads) on the same C5-family rollout, forward and reverse."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _digest(env_extra):
    env = dict(os.environ)
    # the cluster tail kernel (two coarsest levels in one launch, exact
    # coarsest solve) is a different preconditioner, not a plumbing switch:
    # the bitwise comparisons run on the per-level V-cycle
    env["DP_MG_TAIL"] = "0"
    env.update(env_extra)
    out = subprocess.run([sys.executable, os.path.join(HERE, "_variant_run.py")], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("DIGEST")][-1]
    return line.split()[1]


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [{"DP_GRAPHS": "0"}, {"DP_MG_FUSED": "1"}, {"DP_PREJAC": "0"},
                                     {"DP_LS_PRECHECK": "0"}, {"DP_MG_RJ0": "0"}, {"DP_LS_SPECJAC": "0"}],
                         ids=["host-driven-gmres", "fused-coarse-vcycle", "unfused-jacobi0", "no-ls-precheck",
                              "separate-restriction", "no-speculative-trial-jacobian"])
def test_variant_bitwise_identical(variant):
    assert _digest(variant) == _digest({})
