# ncu of every non-evaluation kernel of one C5 csfmm (tree build, traversal/items, upward,
# downward): duration, DRAM bytes and throughput — the HBM-phase evidence of DESIGN.md §3.
# Also the P2M FMA-vs-DMMA A/B.  Usage (under gpurun): bash tools/ncu_hbm.sh TAG
T=${1:-r02}
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size
K='regex:^(?!k_interact|k_mutual|k_dfma).*'
for v in fma dmma; do
  CSFS_B200_P2M=$v timeout 900 ncu --metrics $M --clock-control none -k "$K" --csv --log-file gpurun_out/hbm_${T}_$v.csv python tools/prof_once.py c5 > gpurun_out/hbm_${T}_$v.log 2>&1
  CSFS_B200_P2M=$v timeout 600 python tools/p2m_ab.py $v c5 > gpurun_out/p2m_ab_${T}_$v.json 2> gpurun_out/p2m_ab_${T}_$v.err
done
