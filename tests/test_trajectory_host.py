"""trajectory.csv / forward.json writers (reference cli.py:81-110) - host
logic, no GPU: byte-identical to the reference's csv.writer loop."""
import csv
import io
import json

import numpy as np


def _reference_csv(states):
    """The reference writer (cli.py:92-100), restated with the csv module."""
    f = io.StringIO(newline="")
    f.write("# schema: trajectory v1\n")
    wr = csv.writer(f)
    wr.writerow(["step", "vid", "x", "y", "z"])
    for s, q in enumerate(states):
        pos = q.reshape(-1, 3)
        for vid in range(pos.shape[0]):
            wr.writerow([s, vid] + [f"{c:.17g}" for c in pos[vid]])
    return f.getvalue()


def test_trajectory_csv_bytes_match_reference_writer(tmp_path, rng):
    from paper_2603_16478_b200.trajectory import write_trajectory_csv
    states = [rng.standard_normal(3 * 7) * 10.0 ** rng.integers(-8, 3) for _ in range(4)]
    states[1][2] = -0.0
    states[2][5] = 1e-300
    p = tmp_path / "trajectory.csv"
    write_trajectory_csv(p, states)
    assert p.read_bytes().decode() == _reference_csv(states)


def test_forward_summaries_fields():
    from paper_2603_16478_b200.trajectory import forward_summaries

    class R:
        iterations, converged, residual_history, n_contacts = 7, True, [1e-3, 2e-12], 5
    rows = forward_summaries([R(), R()])
    assert rows[1] == {"step": 2, "iterations": 7, "converged": True, "final_residual": 2e-12, "n_contacts": 5}
    json.dumps(rows)
