# C3 A/B: current vs a previous library build (libvariants/lib_prev.so)
cp paper_2603_16478_b200/libdiffproj_b200.so /tmp/cur.so
run() { timeout 600 python bench.py --config c3 --warmup 3 --skip-insitu --skip-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['e2e']['value'], d['host_syncs_per_step'], sum(d['krylov_iterations']))"; }
for i in 1 2; do
cp libvariants/lib_prev.so paper_2603_16478_b200/libdiffproj_b200.so; run prev
cp /tmp/cur.so paper_2603_16478_b200/libdiffproj_b200.so; run cur
done
