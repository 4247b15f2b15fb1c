#!/bin/bash
# Round-end measurement on one B200 (run under gpurun): bench lines for every
# BASELINE config, the reference arm, the ncu launch list of the default
# bench and `ncu --set full` captures of the hot kernels (each command runs
# once without ncu first).  Outputs go to gpurun_out/<tag>_*;
# tools/ncu_summary.py turns them into markdown / raw pages for profiles/.
set -u
tag=${1:-r2}
out=gpurun_out
mkdir -p $out
run() { name=$1; shift; timeout 600 python bench.py "$@" > $out/${tag}_bench_${name}.json 2> $out/${tag}_bench_${name}.err; echo "$name rc=$?"; tail -1 $out/${tag}_bench_${name}.json | cut -c1-200; }
if [ "${SKIP_BENCH:-0}" != "1" ]; then
run c2 --steps 20 --warmup 5
run c2_bf16 --config c2_bf16 --steps 20 --warmup 5 --no-cpu-baseline
run c3 --config c3 --steps 10 --warmup 3 --no-cpu-baseline
run c4 --config c4 --steps 10 --warmup 3 --no-cpu-baseline
run c5 --config c5 --steps 20 --warmup 5 --no-cpu-baseline
run c1 --config c1 --steps 20 --warmup 5 --no-cpu-baseline
run c2_dense --kind dense --steps 20 --warmup 5 --no-cpu-baseline
run c2_bh --kind bh --steps 20 --warmup 5 --no-cpu-baseline
run c2_ts --steps 10 --warmup 3 --no-cpu-baseline --table-sharded 1
run reference --impl reference --steps 5 --warmup 2
fi
# launch list of the default bench (cold, serialised: shares only)
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $out/${tag}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/${tag}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $out/${tag}_ncu_launches.log 2>&1
echo "launches rc=$?"
# full captures: hash K1f + gather (c2), gather c3, the small-batch kernel
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"hash_sf|gather_row" -s 2 -c 2 \
  -o $out/${tag}_prof -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $out/${tag}_ncu_prof.log 2>&1
echo "prof rc=$?"
python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > $out/${tag}_plain_c3.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"hash_sf|gather_row" -s 2 -c 2 \
  -o $out/${tag}_prof_c3 -f python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > $out/${tag}_ncu_c3.log 2>&1
echo "prof c3 rc=$?"
python tools/small_once.py 1 64 > $out/${tag}_plain_small.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:forward_small -s 2 -c 2 \
  -o $out/${tag}_prof_small -f python tools/small_once.py 1 64 > $out/${tag}_ncu_small.log 2>&1
echo "prof small rc=$?"
python bench.py --kind bh --steps 1 --warmup 3 --no-cpu-baseline > $out/${tag}_plain_bh.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hash_bh64 -s 2 -c 1 \
  -o $out/${tag}_prof_bh -f python bench.py --kind bh --steps 1 --warmup 3 --no-cpu-baseline > $out/${tag}_ncu_bh.log 2>&1
echo "prof bh rc=$?"
# summaries on the box (the .ncu-rep files exceed gpurun's copy-back limit)
python tools/ncu_summary.py launches $out/${tag}_launches.csv > $out/${tag}_launches.md 2>&1
for r in prof prof_c3 prof_small prof_bh; do
  python tools/ncu_summary.py full $out/${tag}_$r.ncu-rep > $out/${tag}_$r.md 2>&1
  ncu -i $out/${tag}_$r.ncu-rep --page raw --csv > $out/${tag}_$r.raw.csv 2>/dev/null
done
python tools/ncu_summary.py traffic $out/${tag}_prof.ncu-rep c2 > $out/${tag}_traffic_c2.json 2>&1
python tools/ncu_summary.py traffic $out/${tag}_prof_c3.ncu-rep c3 > $out/${tag}_traffic_c3.json 2>&1
rm -f $out/${tag}_*.ncu-rep
gzip -f $out/${tag}_launches.csv $out/${tag}_*.raw.csv
ls -la $out | grep $tag
