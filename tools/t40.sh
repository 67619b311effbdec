# assembly: FP32 block group held as floats (80 instead of 128 registers)
set -x
cp paper_2603_16478_b200/libdiffproj_b200.so /tmp/cur.so
for lib in libvariants/lib_c4.so libvariants/lib_f.so; do cp $lib paper_2603_16478_b200/libdiffproj_b200.so; DP_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_assemble -s 2 -c 6 --csv python bench.py --steps 1 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | grep k_assemble | awk -F'","' -v l=$lib '{s+=$NF; n++} END {print "ASM", l, s/n}'; DP_MG_TAIL=1 timeout 300 python tests/_variant_run.py | grep DIGEST; done
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'])"; }
for i in 1 2; do cp libvariants/lib_c4.so paper_2603_16478_b200/libdiffproj_b200.so; run old; cp libvariants/lib_f.so paper_2603_16478_b200/libdiffproj_b200.so; run new; done
cp /tmp/cur.so paper_2603_16478_b200/libdiffproj_b200.so
