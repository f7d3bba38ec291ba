#!/bin/bash
# iteration: GPU parity tests + dengue / MMM bench (kernel-only lines)
cd "$(dirname "$0")/.."
O=gpurun_out/r3i; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x ${TESTK:+-k "$TESTK"} > $O/tests.log 2>&1; echo "tests exit $?" >> $O/tests.log; tail -3 $O/tests.log
for cfg in ${CFGS:-1 2}; do
  env $ENVS timeout 300 python bench.py --config $cfg --steps 300 --warmup 20 --no-cpu-baseline --no-fp64-probe --no-extra-configs > $O/b$cfg.json 2>$O/b$cfg.err
  python - $cfg $O <<'PY'
import json,sys
try:
    d=json.loads(open(f'{sys.argv[2]}/b{sys.argv[1]}.json').read().strip().splitlines()[-1])
    print(sys.argv[1], d['ms_per_step'], d['kernel_ms'], d['roofline']['frac'], d.get('plan',{}).get('smem_bytes'))
except Exception as e:
    print('FAILED', e, open(f'{sys.argv[2]}/b{sys.argv[1]}.err').read()[-1500:])
PY
done
