"""profiles/r02_bench_c5_launches.md from an ncu launch list of the C5 bench
command (usage: python tools/launch_md.py <launches.csv> <bench.json> <script>)."""
import collections
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from summarize_ncu import launches  # noqa: E402

path, bench, script = sys.argv[1], sys.argv[2], sys.argv[3]
tab = launches(path)
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(float)
tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= mi:
        continue
    v = float(r[mi].replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
                                          "msecond": 1e3}.get(r[ui], 1)
    agg[r[ki].split("(")[0]] += v
    tot += v


def share(pred):
    return 100 * sum(v for k, v in agg.items() if pred(k)) / tot


groups = [("fine-level V-cycle sweeps (TMA bulk-copy ring)",
           "`k_mg_smooth<float,1,0,2>` (residual form) + `<float,1,1,2>` (update form + fused (r,z))",
           lambda k: "k_mg_smooth<float" in k),
          ("V-cycle tail: levels 2-3 in one 16-CTA cluster launch", "`k_mg_tail`", lambda k: "k_mg_tail" in k),
          ("level-1 V-cycle (6,859 block rows)", "`k_mg_smooth<double,8>`, `k_mg_restrict_j0`",
           lambda k: "k_mg_smooth<double" in k or "restrict_j0" in k),
          ("element projections + Hessian blocks", "`k_elements<4,*>`", lambda k: "k_elements" in k),
          ("PCG SpMV with fused p-update (FP32 operator)", "`k_pcg_spmv_p<float>`", lambda k: "k_pcg_spmv_p" in k),
          ("assembly + Galerkin products", "`k_assemble`, `k_mg_galerkin`",
           lambda k: "k_assemble" in k or "galerkin" in k),
          ("PCG x/r update + next Jacobi sweep", "`k_pcg_xr_j0`", lambda k: "k_pcg_xr_j0" in k)]
step = json.load(open(bench))["ms_per_step"]
out = ["# C5 bench command, launch list (round 2 final code)", "",
       "DP_GRAPHS=0 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv python "
       "bench.py --steps 20 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu "
       f"(`{script}`, raw list `r02_bench_c5_launches.csv`).  One full 20-step C5 rollout + reverse sweep, "
       "serialised, caches not flushed.  CUDA graphs off: ncu cannot profile kernel nodes of graphs with "
       "conditional (WHILE) nodes, so the PCG/GMRES loops run host-driven here; the kernels are the same.", "", tab]
rest = 100 - sum(share(g[2]) for g in groups)
out += ["", f"Grouped (share of the {tot / 1e3:.0f} ms of serialised device time = {tot / 20e3:.1f} ms per step; the "
        f"bench runs a step in {step:.1f} ms with graphs on, so the GPU idles for at most a few % of the step - host "
        "round-trips of the Newton / line-search loop are hidden behind the kernels):", "",
        "| group | kernels | share |", "|---|---|---|"]
for name, ks, p in groups:
    out.append(f"| {name} | {ks} | {share(p):.1f}% |")
out.append(f"| residual, true residual, contacts, detection, line-search pre-check, vector ops | | {rest:.1f}% |")
open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                  "r02_bench_c5_launches.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out[-11:]))
