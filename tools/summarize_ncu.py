"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and
optionally a --set full report into markdown for profiles/."""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        v = float(r[mi].replace(",", ""))
        v *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    out = ["| kernel | launches | total ms | avg us | share |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        if t / tot < 0.0005:
            continue
        out.append(f"| `{k}` | {n} | {t / 1e3:.2f} | {t / n:.1f} | {100 * t / tot:.1f}% |")
    out.append(f"\nTotal device time in the captured window: {tot / 1e3:.2f} ms over {sum(a[0] for a in agg.values())} launches.")
    return "\n".join(out)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size"]
    idx = [h.index(w) for w in want if w in h]
    names = [h[i] + (f" ({units[i]})" if units[i] else "") for i in idx]
    out = ["| kernel | " + " | ".join(names) + " |", "|---" * (len(idx) + 1) + "|"]
    for r in rows[2:]:
        out.append(f"| `{r[h.index('Kernel Name')].split('(')[0]}` | " + " | ".join(r[i] for i in idx) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else full(path))
