#!/bin/bash
# Round evidence on one B200: GPU tests, smoke, bench (both arms), slab shapes, ncu launch
# list, ncu full captures of the iteration's kernels (incl. the finalize, with source).
# Outputs under gpurun_out/ (copy the summaries to profiles/).
set -x
TAG=${1:-r2}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 python bench.py --n 256 --no-cpu-baseline > gpurun_out/bench256_$TAG.json 2> gpurun_out/bench256_$TAG.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$TAG.json 2>&1
timeout 400 python tools/slab_shape.py --L 512,256,128,64 --steps 50 --out gpurun_out/slab_shape_$TAG.json > /dev/null 2>&1
nproc > gpurun_out/host_$TAG.txt; lscpu | grep -i "model name" >> gpurun_out/host_$TAG.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_cheb_tb4|k_update_xr2|k_stencil_tma|k_finalize" --launch-skip 24 --launch-count 8 -o gpurun_out/full_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
# summaries on the box (the .ncu-rep files are too large to bring back)
for r in full_$TAG; do
  python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/${r}_summary.txt 2>&1
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page source --csv -k regex:k_finalize > gpurun_out/${r}_finalize_source.csv 2>/dev/null
  rm -f gpurun_out/$r.ncu-rep
done
ls -la gpurun_out
