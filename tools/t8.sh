cp paper_2603_16478_b200/libdiffproj_b200.so /tmp/orig.so
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-insitu --skip-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['e2e']['value'])"; }
for i in 1 2; do
cp libvariants/lib_trig0.so paper_2603_16478_b200/libdiffproj_b200.so; DP_PDL=1 run trig0
cp libvariants/lib_trig1.so paper_2603_16478_b200/libdiffproj_b200.so; DP_PDL=1 run trig1
DP_PDL=0 run off
done
cp /tmp/orig.so paper_2603_16478_b200/libdiffproj_b200.so
