timeout 400 python bench.py > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k "regex:k_assemble|k_elements" -s 20 -c 12 --csv python bench.py --steps 1 --warmup 3 --warmup-seconds 0 --skip-e2e --skip-cpu > gpurun_out/s_ncu.csv 2>&1
