set -x
for L in base new; do
  if [ $L = base ]; then export BCGS_LIB=$PWD/paper_2503_08935_b200/lib/libbcgs_base.so; else unset BCGS_LIB; fi
  python tools/tb_bench.py --n 512 --degree 4 --variants 7 2>&1 | tail -3
  python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', d['ms_per_step'], d['kernel_ms_per_step'], d['clocks'])"
done
