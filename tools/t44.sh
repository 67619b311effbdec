# L1::no_allocate loads in the residual gather and the assembly: kernel times, digest, A/B
set -x
cp paper_2603_16478_b200/libdiffproj_b200.so /tmp/cur.so
for lib in libvariants/lib_a.so libvariants/lib_na2.so; do cp $lib paper_2603_16478_b200/libdiffproj_b200.so; DP_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_residual|k_assemble" -s 5 -c 20 --csv python bench.py --steps 1 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | grep -E "k_residual|k_assemble" | awk -F'","' -v l=$lib '{split($5,a,"("); k=a[1]; s[k]+=$NF; n[k]++} END {for (k in s) print "KT", l, k, s[k]/n[k]}'; DP_MG_TAIL=1 timeout 300 python tests/_variant_run.py | grep DIGEST; done
run() { timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'])"; }
for i in 1 2; do cp libvariants/lib_a.so paper_2603_16478_b200/libdiffproj_b200.so; run old; cp libvariants/lib_na2.so paper_2603_16478_b200/libdiffproj_b200.so; run new; done
cp /tmp/cur.so paper_2603_16478_b200/libdiffproj_b200.so
