#!/bin/bash
# Tree-build phase of every built variant in _variants/ (GPU box): tools/quick_perf.py
cd "$(dirname "$0")/.."
for so in _variants/*/libcsfs_b200.so; do
  echo "== $so"
  CSFS_B200_LIB=$PWD/$so timeout 300 python tools/quick_perf.py "$@" 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        if d['it']==2: print('  %s tree %.5f lists %.5f total %.4f'%(d['cfg'],d['t_tree_build'],d['t_lists'],d['t_total']))
"
done
