#!/bin/bash
# Round-2 evidence (writes gpurun_out/): the default bench line (config 4 tree-OMP),
# every config's line, the config-4 launch list with DRAM bytes, ncu --set full
# captures of the dominant kernels.
mkdir -p gpurun_out
B="python bench.py"
timeout 900 $B > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err
timeout 2400 bash tools/all_configs.sh > gpurun_out/r02_all_configs.log 2>&1
cp gpurun_out/configs.jsonl gpurun_out/r02_all_configs.jsonl
Q="--profile-run --steps 1 --warmup 1"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 400 --csv --log-file gpurun_out/r02_c4_launches.csv $B $Q > gpurun_out/ncu_list.log 2>&1
NCU="timeout 900 ncu --set full --import-source on --clock-control none"
$NCU -k regex:update_wide_kernel -s 6 -c 1 -o gpurun_out/r02_full_update_wide_c4 $B $Q > gpurun_out/ncu_u.log 2>&1
$NCU -k regex:score_st_kernel -s 20 -c 1 -o gpurun_out/r02_full_score_st_c4 $B $Q > gpurun_out/ncu_s.log 2>&1
ls -la gpurun_out
