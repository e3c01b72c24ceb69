# A/B of library variants built under _variants/<name>/libcsfs_b200.so (see tools/variant_accuracy.py)
for so in _variants/*/libcsfs_b200.so paper_2508_13550_b200/libcsfs_b200.so; do echo "== $so"; for rep in 1 2; do CSFS_B200_LIB=$PWD/$so timeout 300 python tools/quick_perf.py ${AB_CFG:-c5} 2>&1 | grep '"it": 2' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  %s total %.4f interact %.4f'%(d['cfg'],d['t_total'],d['t_interact']))"; done; done
