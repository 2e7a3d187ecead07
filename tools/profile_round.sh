#!/bin/bash
# Round evidence: bench lines (ours + reference arm, every config), the c1 launch list
# with DRAM bytes, and ncu --set full captures of the dominant kernels.  Writes gpurun_out/.
mkdir -p gpurun_out
B="python bench.py"
timeout 600 $B > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 $B --impl reference --steps 3 --warmup 3 > gpurun_out/bench_c1_ref.json 2> gpurun_out/bench_c1_ref.err
timeout 1500 bash tools/all_configs.sh > gpurun_out/all_configs.log 2>&1
Q="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 400 --csv --log-file gpurun_out/c1_launches.csv $B $Q > gpurun_out/ncu_list.log 2>&1
NCU="timeout 600 ncu --set full --import-source on --clock-control none"
$NCU -k regex:update_omp8_kernel -s 4 -c 1 -o gpurun_out/full_update $B $Q > gpurun_out/ncu_u.log 2>&1
$NCU -k regex:score_ts_kernel -s 4 -c 1 -o gpurun_out/full_score_ts $B $Q > gpurun_out/ncu_s.log 2>&1
$NCU -k regex:scatter_scan_kernel -s 3 -c 1 -o gpurun_out/full_scatter $B $Q > gpurun_out/ncu_sc.log 2>&1
$NCU -k regex:score_st_kernel -s 3 -c 1 -o gpurun_out/full_score_st $B --config 2 $Q > gpurun_out/ncu_st.log 2>&1
$NCU -k regex:exact_scan_kernel -s 2 -c 1 -o gpurun_out/full_exact $B --config 4 --selector exact --patches 8192 $Q \
  > gpurun_out/ncu_x.log 2>&1
ls -la gpurun_out
