set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "segment" > gpurun_out/s6_pytest_seg.log 2>&1; tail -n 3 gpurun_out/s6_pytest_seg.log
timeout 1300 python -m pytest tests -m gpu -x -q > gpurun_out/s6_pytest.log 2>&1; tail -n 3 gpurun_out/s6_pytest.log
