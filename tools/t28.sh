# variance of the driver's C5 command on one box (3 back-to-back runs, final code) + GPU tests
set -x
for i in 1 2 3; do timeout 500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/t28_$i.json 2> gpurun_out/t28_$i.err; done
python - <<'PY'
import json
rs=[json.load(open(f"gpurun_out/t28_{i}.json")) for i in (1,2,3)]
out=dict(command="python bench.py --gpus 1 --steps 20 --warmup 5 (x3, one box, back to back)",
         value=[r["value"] for r in rs], e2e=[r["e2e"]["value"] for r in rs],
         roofline_frac=[r["roofline"]["frac"] for r in rs], clocks=[r["clocks"] for r in rs],
         host_syncs_per_step=[r["host_syncs_per_step"] for r in rs], gpu_launches=[r["gpu_launches"] for r in rs])
json.dump(out, open("gpurun_out/t28_repeats.json","w"), indent=1)
print("REPEATS", out["value"], out["e2e"], out["roofline_frac"])
PY
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t28_gputests.log 2>&1; tail -2 gpurun_out/t28_gputests.log
