# restriction with 8-lane groups per coarse row (+ Minv prefetch): variants bitwise, A/B vs previous build
set -x
timeout 1200 python -m pytest tests/test_gpu_variants.py -x -q > gpurun_out/t35_var.log 2>&1; tail -2 gpurun_out/t35_var.log
cp paper_2603_16478_b200/libdiffproj_b200.so /tmp/cur.so
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], sum(d['krylov_iterations']), d['adjoint_krylov_iterations'], sum(d['newton_iterations']))"; }
for i in 1 2; do
cp libvariants/lib_prev.so paper_2603_16478_b200/libdiffproj_b200.so; run prev
cp /tmp/cur.so paper_2603_16478_b200/libdiffproj_b200.so; run cur
done
