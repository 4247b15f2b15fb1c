set -u
out=gpurun_out; mkdir -p $out
python -m pytest tests/test_gpu_group.py tests/test_table_slices.py -m gpu -q -x > $out/t4_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $out/t4_pytest.log
python tools/hash_sweep.py c2 c3 c4 2>&1 | tee $out/t4_hash_sweep.txt
python tools/gather_sweep.py c2 c2_bf16 c3 c4 --variants 0,1 2>&1 | tee $out/t4_gather_sweep.txt
timeout 900 python bench.py --table-sharded 1 --no-cpu-baseline --steps 10 > $out/t4_bench_ts.json 2> $out/t4_bench_ts.err; echo "bench ts rc=$?"; python -c "import json;d=json.loads(open('$out/t4_bench_ts.json').read().strip().splitlines()[-1]);print(json.dumps(d.get('table_sharded'),indent=1))"; tail -3 $out/t4_bench_ts.err
python tools/hash_sweep.py c2 --reps 1 > $out/t4_plain.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:hash_sf -s 1 -c 1 -o $out/t4_hash -f python tools/hash_sweep.py c2 --reps 1 > $out/t4_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $out/t4_hash.ncu-rep --page raw --csv > $out/t4_hash_raw.csv 2>/dev/null; ncu -i $out/t4_hash.ncu-rep --page source --csv > $out/t4_hash_source.csv 2>/dev/null; ncu -i $out/t4_hash.ncu-rep --page details --csv > $out/t4_hash_details.csv 2>/dev/null; rm -f $out/t4_hash.ncu-rep; gzip -f $out/t4_hash_*.csv; ls -la $out | tail -5
