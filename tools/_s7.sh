set -x
timeout 1300 python -m pytest tests -m gpu -x -q > gpurun_out/s7_pytest.log 2>&1; tail -n 3 gpurun_out/s7_pytest.log
timeout 300 python tools/slab_shape.py --n 512 --L 512,64 --pdl 0,1 --steps 50 > gpurun_out/s7_slab.txt 2>&1
timeout 300 python tools/slab_shape.py --n 256 --L 256 --pdl 0,1 --steps 100 >> gpurun_out/s7_slab.txt 2>&1
timeout 300 python tools/slab_shape.py --n 64 --L 64 --pdl 0,1 --steps 500 >> gpurun_out/s7_slab.txt 2>&1
timeout 400 python bench.py > gpurun_out/s7_bench.json 2> gpurun_out/s7_bench.err
