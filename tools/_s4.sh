set -x
timeout 1300 python -m pytest tests -m gpu -x -q > gpurun_out/s4_pytest.log 2>&1; tail -n 3 gpurun_out/s4_pytest.log
timeout 300 python tools/slab_shape.py --L 512,64 --steps 30 > gpurun_out/s4_slab.txt 2>&1
