set -x
for v in 7 8 10; do
  BCGS_LIB=scratch/xp/libbcgs.so timeout 300 ncu --set full --clock-control none -k regex:"k_cheb" --launch-skip 3 --launch-count 1 -o gpurun_out/xp_v$v python tools/tb_bench.py --n 512 --degree 4 --variants $v > gpurun_out/xp_v$v.log 2>&1
  python tools/ncu_summary.py gpurun_out/xp_v$v.ncu-rep > gpurun_out/xp_v${v}_summary.txt 2>&1
  rm -f gpurun_out/xp_v$v.ncu-rep
done
BCGS_LIB=scratch/xp/libbcgs.so timeout 300 python tools/tb_bench.py --n 512 --degree 4 --variants 7,8,10 > gpurun_out/xp_tb.txt 2>&1
