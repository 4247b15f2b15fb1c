#!/bin/bash
# Round-end measurement on one B200 (run under gpurun): bench lines for every
# BASELINE config, the reference arm, the ncu launch list of the default
# bench and `ncu --set full` captures of the hot kernels.  Outputs go to
# gpurun_out/<tag>_*; tools/ncu_summary.py turns them into profiles/.
set -u
tag=${1:-r1}
out=gpurun_out
mkdir -p $out
run() { name=$1; shift; timeout 300 python bench.py "$@" > $out/${tag}_bench_${name}.json 2> $out/${tag}_bench_${name}.err; echo "$name rc=$?"; tail -1 $out/${tag}_bench_${name}.json | cut -c1-200; }
run c2 --steps 20 --warmup 5
run c2_bf16 --config c2_bf16 --steps 20 --warmup 5 --no-cpu-baseline
run c3 --config c3 --steps 10 --warmup 3 --no-cpu-baseline
run c4 --config c4 --steps 10 --warmup 3 --no-cpu-baseline
run c5 --config c5 --steps 20 --warmup 5 --no-cpu-baseline
run c1 --config c1 --steps 20 --warmup 5 --no-cpu-baseline
run c2_dense --kind dense --steps 20 --warmup 5 --no-cpu-baseline
run c2_bh --kind bh --steps 20 --warmup 5 --no-cpu-baseline
run c3_table --config c3 --shard table --steps 10 --warmup 3 --no-cpu-baseline
run reference --impl reference --steps 3 --warmup 3
for k in signflip dense acdc bh; do timeout 300 python tools/backward_time.py c2 $k >> $out/${tag}_backward.txt 2>&1; done
tail -4 $out/${tag}_backward.txt
# launch list of the default bench (cold, serialised: shares only)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/${tag}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $out/${tag}_ncu_launches.log 2>&1
echo "launches rc=$?"
# full captures: hash + gather (c2 signflip), dense tcgen05 (c2 dense), gather c4
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"hash_structured|gather_row" -s 2 -c 2 \
  -o $out/${tag}_prof -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $out/${tag}_ncu_prof.log 2>&1
echo "prof rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"dense_tcgen05|dense_split|dense_fixup" -s 3 -c 3 \
  -o $out/${tag}_prof_dense -f python bench.py --kind dense --steps 1 --warmup 3 --no-cpu-baseline > $out/${tag}_ncu_dense.log 2>&1
echo "prof dense rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gather_row" -s 1 -c 1 \
  -o $out/${tag}_prof_c4 -f python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > $out/${tag}_ncu_c4.log 2>&1
echo "prof c4 rc=$?"
# summaries on the box (the .ncu-rep files together exceed gpurun's 64 MiB
# copy-back limit): markdown + raw CSV pages, then keep only the c2 capture
python tools/ncu_summary.py launches $out/${tag}_launches.csv > $out/${tag}_launches.md 2>&1
for r in prof prof_dense prof_c4; do
  python tools/ncu_summary.py full $out/${tag}_$r.ncu-rep > $out/${tag}_$r.md 2>&1
  ncu -i $out/${tag}_$r.ncu-rep --page raw --csv > $out/${tag}_$r.raw.csv 2>/dev/null
done
python tools/ncu_summary.py traffic $out/${tag}_prof.ncu-rep c2 > $out/${tag}_traffic_c2.json 2>&1
python tools/ncu_summary.py traffic $out/${tag}_prof_c4.ncu-rep c4 > $out/${tag}_traffic_c4.json 2>&1
rm -f $out/${tag}_prof_dense.ncu-rep $out/${tag}_prof_c4.ncu-rep
gzip -f $out/${tag}_launches.csv $out/${tag}_*.raw.csv
