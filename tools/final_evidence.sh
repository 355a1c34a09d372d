#!/bin/bash
# On the GPU box: the round's evidence in one call -- bench lines of every
# config (ours, then the reference arm), the ncu launch list of the default
# bench command, per-config ncu metric evidence (profiles/evidence_configN.json)
# and full ncu captures of the top kernels (K1 on config 2, the K2 filter on
# config 4).  Everything lands in gpurun_out/final_* (copy what is judged to
# profiles/).
#   tools/final_evidence.sh [configs...]      (default: 2 1 3 4 5)
cd "$(dirname "$0")/.."
CFGS=${*:-2 1 3 4 5}
mkdir -p gpurun_out
for c in $CFGS; do
  timeout 600 python bench.py --config "$c" --steps 20 --warmup 3 > gpurun_out/final_bench_c$c.jsonl 2> gpurun_out/final_bench_c$c.err
done
for c in $CFGS; do
  timeout 600 python bench.py --impl reference --config "$c" --steps 3 --warmup 1 > gpurun_out/final_ref_c$c.jsonl 2> gpurun_out/final_ref_c$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 \
  --csv --log-file gpurun_out/final_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/final_launches_c2.log 2>&1
timeout 1500 tools/evidence.sh $CFGS > gpurun_out/final_evidence.log 2>&1
cp profiles/evidence_config*.json gpurun_out/ 2>/dev/null
timeout 600 ncu --set full --import-source on --clock-control none -k regex:csr4 -s 2 -c 1 -o gpurun_out/final_csr4_c2 -f \
  python tools/ncu_target.py --config 2 > gpurun_out/final_ncu_csr4.log 2>&1
ncu -i gpurun_out/final_csr4_c2.ncu-rep --page details --csv > gpurun_out/final_csr4_c2_details.csv 2>/dev/null
ncu -i gpurun_out/final_csr4_c2.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/final_csr4_c2_src.csv 2>/dev/null
timeout 600 ncu --set full --import-source on --clock-control none -k regex:elem_filter -s 1 -c 1 -o gpurun_out/final_filter_c4 -f \
  python tools/ncu_target.py --config 4 > gpurun_out/final_ncu_filter.log 2>&1
ncu -i gpurun_out/final_filter_c4.ncu-rep --page details --csv > gpurun_out/final_filter_c4_details.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep  # large; the csv pages above are what is kept
echo done
