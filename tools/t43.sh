# residual gather: element-force loads without L1 allocation (DP_RES_NA)
set -x
cp paper_2603_16478_b200/libdiffproj_b200.so /tmp/cur.so
for lib in libvariants/lib_a.so libvariants/lib_na.so; do cp $lib paper_2603_16478_b200/libdiffproj_b200.so; DP_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_residual -s 5 -c 10 --csv python bench.py --steps 1 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu 2>/dev/null | grep k_residual | awk -F'","' -v l=$lib '{s+=$NF; n++} END {print "RES", l, s/n}'; done
cp /tmp/cur.so paper_2603_16478_b200/libdiffproj_b200.so
