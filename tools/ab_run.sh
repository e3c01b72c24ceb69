# A/B of the _variants/ libraries on the GPU box: timing (tools/ab_variants.sh) per config,
# then full-size parity against the reference (tools/variant_parity.py).
# Usage: bash tools/ab_run.sh TAG "c5 c3" "c5"
set -x
T=$1
mkdir -p gpurun_out
for c in $2; do AB_CFG=$c timeout 900 bash tools/ab_variants.sh >> gpurun_out/ab_$T.log 2>&1; done
[ -n "$3" ] && timeout 2400 python tools/variant_parity.py $3 > gpurun_out/variant_parity_$T.log 2>&1
echo done
