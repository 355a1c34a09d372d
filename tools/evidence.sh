#!/bin/bash
# On the GPU box: ncu metric capture of tools/ncu_target.py for the given
# configs, joined into profiles/evidence_configN.json (read by bench.py).
#   tools/evidence.sh 1 2 3
set -e
cd "$(dirname "$0")/.."
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio
M=$M,dram__bytes_read.sum,dram__bytes_write.sum
M=$M,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
M=$M,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active
M=$M,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
M=$M,sm__warps_active.avg.pct_of_peak_sustained_active
mkdir -p gpurun_out
for c in "$@"; do
  python tools/ncu_target.py --config "$c" > /dev/null  # exits 0 without ncu first
  ncu --metrics "$M" --clock-control none --csv --log-file gpurun_out/evidence_c$c.csv \
      python tools/ncu_target.py --config "$c" > gpurun_out/evidence_c$c.log 2>&1
  python tools/make_evidence.py --config "$c" --csv gpurun_out/evidence_c$c.csv \
      --target gpurun_out/target_config$c.json --tag r02
done
