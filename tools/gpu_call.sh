set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/t2_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/t2_pytest.log
timeout 600 python bench.py > gpurun_out/t2_bench.json 2> gpurun_out/t2_bench.err; echo "bench rc=$?"; cut -c1-3000 gpurun_out/t2_bench.json
timeout 900 python bench.py --table-sharded 1 --no-cpu-baseline --steps 10 > gpurun_out/t2_bench_ts.json 2> gpurun_out/t2_bench_ts.err; echo "bench ts rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/t2_bench_ts.json').read().strip().splitlines()[-1]);print(json.dumps(d.get('table_sharded'),indent=1))"; tail -3 gpurun_out/t2_bench_ts.err
./tools/microbench/l2probe quick > gpurun_out/l2probe_q.log 2>&1 && ncu --set full --clock-control none -o gpurun_out/l2probe -f ./tools/microbench/l2probe quick > gpurun_out/l2probe_ncu.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/l2probe.ncu-rep --page raw --csv > gpurun_out/l2probe_raw.csv 2>/dev/null; rm -f gpurun_out/l2probe.ncu-rep; gzip -f gpurun_out/l2probe_raw.csv; ls -la gpurun_out
