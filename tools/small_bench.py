"""Per-iteration time of small configs with / without CUDA-graph replay (launch-bound regime).
python tools/small_bench.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth_inputs as si  # noqa: E402
from paper_2503_08935_b200 import bcgs  # noqa: E402

for n, pc, k in [(32, "none", 0), (32, "gnocomm", 4), (64, "gnocomm", 4), (128, "gnocomm", 4),
                 (256, "gnocomm", 4)]:
    row = []
    for graph in (0, 1):
        s = bcgs.Solver(n, si.unit_cube_h(n))
        s.set_option(bcgs.OPT_GRAPH, graph)
        s.set_preconditioner(pc, k)
        s.set_rhs_random(si.SEED)
        s.begin(fixed_iters=1200)
        s.iterate(100)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.iterate(1000)
        torch.cuda.synchronize()
        row.append((time.perf_counter() - t0) / 1000 * 1e6)
        s.close()
    print(f"{n}^3 {pc} k={k}: {row[0]:.1f} us/iter direct, {row[1]:.1f} us/iter graph", flush=True)
