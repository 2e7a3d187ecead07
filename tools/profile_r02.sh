#!/bin/bash
# Round-2 evidence (writes gpurun_out/): the default bench line (config 4 tree-OMP)
# and its reference arm, every config's line, warm per-launch durations, the
# config-4 launch list with DRAM bytes, ncu --set full captures of the dominant
# kernels, the GPU test log.  Every profiled command first runs to completion
# without ncu.  Summaries for profiles/: tools/ncu_summary.py, tools/traffic.py.
mkdir -p gpurun_out
B="python bench.py"
timeout 900 $B > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; echo bench rc=$?
timeout 600 $B --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_c4_reference.json 2> gpurun_out/r02_bench_ref.err
timeout 2400 bash tools/all_configs.sh > gpurun_out/r02_all_configs.log 2>&1; cp gpurun_out/configs.jsonl gpurun_out/r02_all_configs.jsonl
KPROF_LIST=1 timeout 300 python tools/kprof.py 4 524288 2>&1 | grep -v -i warn > gpurun_out/r02_kprof_c4.txt
Q="--profile-run --steps 1 --warmup 1"
timeout 600 $B $Q > gpurun_out/profile_run_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 400 --csv --log-file gpurun_out/r02_c4_step_launches.csv $B $Q > gpurun_out/ncu_list.log 2>&1
NCU="timeout 900 ncu --set full --import-source on --clock-control none -f"
$NCU -k regex:score_sh_kernel -s 30 -c 2 -o gpurun_out/r02_full_score_sh_c4 $B $Q > gpurun_out/ncu_s.log 2>&1
$NCU -k regex:update_gram_kernel -s 17 -c 1 -o gpurun_out/r02_full_update_gram_c4 $B $Q > gpurun_out/ncu_u.log 2>&1
$NCU -k regex:gram_corr_kernel -s 32 -c 2 -o gpurun_out/r02_full_gram_corr_c4 $B $Q > gpurun_out/ncu_c.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_pytest_gpu.log 2>&1
tail -1 gpurun_out/r02_pytest_gpu.log
timeout 120 tools/_stream_bench > gpurun_out/r02_stream_bench.txt 2>&1
CFG=4 timeout 600 python tools/e2e_sweep.py 65536 131072 262144 524288 2>&1 | grep -v -i warn > gpurun_out/r02_e2e_sweep_c4.txt
