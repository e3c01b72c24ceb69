#!/bin/bash
# Run tools/quick_perf.py against every built variant in _variants/ (GPU box).
cd "$(dirname "$0")/.."
for so in _variants/*/libcsfs_b200.so; do
  echo "== $so"
  CSFS_B200_LIB=$PWD/$so timeout 300 python tools/quick_perf.py "$@" 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        if d['it']==2: print('  %s interact %.4f s  total %.4f s  evals/s %.3e'%(d['cfg'],d['t_interact'],d['t_total'],d['evals_per_s']))
    else: print(l.rstrip())
"
done
