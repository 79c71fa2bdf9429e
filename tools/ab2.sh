for L in base new; do
  if [ $L = base ]; then export BCGS_LIB=$PWD/paper_2503_08935_b200/lib/libbcgs_base.so; else unset BCGS_LIB; fi
  python tools/mp_bench.py --n 512 --degrees 8,24 --reps 3 2>&1 | sed "s/^/$L /"
  python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'])"
done
