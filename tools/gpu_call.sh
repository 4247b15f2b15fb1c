#!/bin/bash
# One gpurun call: GPU tests, bench lines for the BASELINE configs, optional
# extra command.  Usage: bash tools/gpu_call.sh <tag> [pytest-args]
set -u
tag=${1:-t}
shift || true
out=gpurun_out
mkdir -p $out
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > $out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -8 $out/${tag}_pytest.log
fi
run() { name=$1; shift; timeout 600 python bench.py "$@" > $out/${tag}_bench_${name}.json 2> $out/${tag}_bench_${name}.err; echo "$name rc=$?";
  python - "$out/${tag}_bench_${name}.json" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r=d.get('roofline',{})
    print(f"  value={d['value']/1e6:.3f}M ms={d['ms_per_step']} stages={d.get('stages_ms')} frac={r.get('frac')} frac_fwd={r.get('frac_forward')} e2e={d['e2e']['value']/1e6:.3f}M launches={d.get('gpu_launches')} clocks={d.get('clocks',{}).get('sm_mhz')}")
    if 'table_sharded' in d: print('  ts', json.dumps(d['table_sharded'])[:1500])
    if 'small_batch_latency' in d: print('  small', d['small_batch_latency'])
    if 'cpu_baseline' in d: print('  cpu', d['cpu_baseline'].get('value'))
except Exception as e:
    print('  parse error', e); print(open(sys.argv[1]).read()[-1500:])
PY
  tail -2 $out/${tag}_bench_${name}.err; }
for c in ${BENCH_CONFIGS:-c2 c2_bf16 c3 c4 c5}; do
  if [ "$c" = "c2" ]; then run c2 --steps 20 --warmup 5; else run $c --config $c --steps 20 --warmup 5 --no-cpu-baseline; fi
done
if [ -n "${EXTRA:-}" ]; then bash -c "$EXTRA"; fi
