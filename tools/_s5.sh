set -x
strings paper_2503_08935_b200/lib/libbcgs.so | grep -c 'tb schedule'
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "segment or variants_bitwise or stencil_tma or xpair" > gpurun_out/s5_pytest.log 2>&1; tail -n 3 gpurun_out/s5_pytest.log
timeout 300 python tools/slab_shape.py --n 256 --L 256 --schedule 1,2,0 --steps 50 > gpurun_out/s5_slab.txt 2>&1
timeout 300 python tools/slab_shape.py --n 512 --L 512,64 --schedule 0,2 --steps 30 >> gpurun_out/s5_slab.txt 2>&1
timeout 400 python bench.py > gpurun_out/s5_bench.json 2> gpurun_out/s5_bench.err
