# Round-2 artefacts: the driver's bench command, the reference arm, the GPU
# tests, the warm launch list of the bench command (graphs off so ncu can see
# the kernels) and one --set full capture of the dominant kernel.
set -x
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/f2_ref.json 2> gpurun_out/f2_ref.err
for c in c1 c3 c4; do python bench.py --config $c --warmup 3 --skip-insitu > gpurun_out/f2_$c.json 2> gpurun_out/f2_$c.err; done
DP_GRAPHS=0 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/f2_launches.csv python bench.py --steps 20 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu \
  > gpurun_out/f2_ncu.log 2>&1
DP_GRAPHS=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mg_smooth -s 220 -c 2 \
  -o gpurun_out/f2_smooth python bench.py --steps 3 --warmup 0 --warmup-seconds 0 --skip-cpu --skip-e2e --skip-insitu \
  > gpurun_out/f2_ncu_full.log 2>&1
nproc > gpurun_out/f2_nproc.txt; lscpu | grep "Model name" >> gpurun_out/f2_nproc.txt
