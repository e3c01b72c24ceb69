#!/bin/bash
# Build libcsfs_b200 variants of the evaluation kernel's tuning knobs into _variants/<name>/
set -e
cd "$(dirname "$0")/.."
for v in "$@"; do
  name=$(echo "$v" | sed 's/-DCSFS_//g' | tr ' =' '_-')
  out=_variants/$name
  mkdir -p $out/obj
  make -s -C paper_2508_13550_b200/csrc OUT=$PWD/$out/libcsfs_b200.so OBJ=$PWD/$out/obj EXTRA_NVFLAGS="$v" -j8 >/dev/null
  echo "$out/libcsfs_b200.so"
done
