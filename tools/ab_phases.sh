# A/B of _variants/*/libcsfs_b200.so and the in-tree library: median phase times (ms)
for so in _variants/*/libcsfs_b200.so paper_2508_13550_b200/libcsfs_b200.so; do
  for c in ${AB_CFGS:-c5}; do echo "$so $(CSFS_B200_LIB=$PWD/$so timeout 300 python tools/phase_ab.py $c 2>&1 | tail -1)"; done
done
