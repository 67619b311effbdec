# A/B of the cluster tail kernel (DP_MG_TAIL) on C5; phase timings with DP_MG_TAIL_DBG
mkdir -p gpurun_out
DP_MG_TAIL=1 DP_MG_TAIL_DBG=1 DP_GRAPHS=0 timeout 300 python bench.py --gpus 1 --steps 3 --warmup 3 --skip-insitu --skip-e2e --skip-cpu > gpurun_out/tdbg.json 2> gpurun_out/tdbg.err; grep "tail phases" gpurun_out/tdbg.err | tail -1
for t in 0 1 0 1; do DP_MG_TAIL=$t timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-insitu 2>gpurun_out/ab_err_$t.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TAIL', $t, d['value'], d['e2e']['value'], d['ms_per_step'])"; done
