#!/bin/bash
# Round evidence: bench lines (ours + reference arm), the c1 launch list with DRAM
# bytes, and ncu --set full captures of the dominant kernels.  Writes gpurun_out/.
set -x
mkdir -p gpurun_out
B="python bench.py"
timeout 600 $B > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 $B --impl reference --steps 3 --warmup 3 > gpurun_out/bench_c1_ref.json 2> gpurun_out/bench_c1_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 400 --csv --log-file gpurun_out/c1_launches.csv $B --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_list.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:update_omp8_kernel -s 12 -c 1 \
  -o gpurun_out/full_update $B --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_u.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:score_ts_kernel -s 37 -c 1 \
  -o gpurun_out/full_score_ts $B --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_s.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:score_st_kernel -s 3 -c 1 \
  -o gpurun_out/full_score_st $B --config 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_st.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:exact_scan_kernel -s 2 -c 1 \
  -o gpurun_out/full_exact $B --config 4 --selector exact --patches 8192 --steps 1 --warmup 1 --no-e2e \
  --no-cpu-baseline > gpurun_out/ncu_x.log 2>&1
ls -la gpurun_out
