set -x
strings paper_2503_08935_b200/lib/libbcgs.so | grep 'temporally blocked layout'
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "variants_bitwise or xpair or stencil_tma" > gpurun_out/s3_pytest.log 2>&1; tail -n 3 gpurun_out/s3_pytest.log
timeout 300 python tools/tb_bench.py --n 512 --degree 4 --variants 7,8,10 --oracle > gpurun_out/s3_tb.txt 2>&1
timeout 300 python tools/slab_shape.py --L 512,256,128,64 --stencil 1,32 --steps 30 > gpurun_out/s3_slab.txt 2>&1
timeout 200 python tools/slab_shape.py --L 64 --stencil 8,16,22 --steps 30 >> gpurun_out/s3_slab.txt 2>&1
