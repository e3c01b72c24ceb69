for so in _variants/*/libcsfs_b200.so; do echo "== $so"; CSFS_B200_LIB=$PWD/$so timeout 300 python tools/quick_perf.py c5 c3 2>&1 | grep '"it": 2' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  %s total %.4f down %.5f up %.5f'%(d['cfg'],d['t_total'],d['t_downward'],d['t_upward']))"; done
