#!/bin/bash
# Round-2 measurement set: bench (both arms), TF32 peak, configs 4/5, ncu
# captures (config-1 GEMM/CSC/aggregate, config-3 ranking, config-4 CSC/
# aggregate/GEMM DRAM traffic). Each ncu runs only after its command exits 0;
# reports are reduced to CSV on the box (raw metrics + source hot spots).
TAG=${1:-r2p}
O=gpurun_out
summarize() {   # $1 = report base name
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>/dev/null
  ncu -i $O/$1.ncu-rep --page details --csv > $O/$1_details.csv 2>/dev/null
  sz=$(stat -c %s $O/$1.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -gt 12000000 ]; then rm -f $O/$1.ncu-rep; fi
}
if [ -z "$SKIP_BENCH" ]; then
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err; echo ref rc=$?
timeout 300 python tools/tf32_peak.py > $O/${TAG}_tf32_peak.json 2>&1; echo tf32 rc=$?
timeout 900 python tools/bench_config4.py --config 4 > $O/${TAG}_config4.json 2> $O/${TAG}_config4.err; echo c4 rc=$?
timeout 900 python tools/bench_config4.py --config 5 > $O/${TAG}_config5.json 2> $O/${TAG}_config5.err; echo c5 rc=$?
fi
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_umma_packed|k_csc_backward|k_csc_dots|k_aggregate" \
  -s 40 -c 8 -o $O/${TAG}_c1_full $CMD > $O/${TAG}_c1_ncu.log 2>&1; echo ncu c1 rc=$?; summarize ${TAG}_c1_full
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rank_umma" -c 2 \
  -o $O/${TAG}_eval_full python tools/eval_bench.py > $O/${TAG}_eval_ncu.log 2>&1; echo ncu eval rc=$?; summarize ${TAG}_eval_full
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_csc_backward|k_aggregate|k_umma_packed" -c 6 \
  -o $O/${TAG}_c4_full python tools/bench_config4.py --config 4 --rounds 1 > $O/${TAG}_c4_ncu.log 2>&1; echo ncu c4 rc=$?; summarize ${TAG}_c4_full
du -sh $O
