"""CPU checks of bench.py's host-side bookkeeping (no GPU): BASELINE.json config names, the
algorithmic-byte model, the measured-peak lookup and the FP64 flop model of the blocked
Chebyshev kernels."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_workload_labels_follow_baseline_configs():
    b = load_bench()
    assert b.workload(512, "gnocomm", 4) == "C3 512^3 GNoComm(CI) k=4"
    assert b.workload(256, "gnocomm", 4).startswith("C2 256^3")
    assert b.workload(1024, "gnocomm", 4).startswith("C5 1024^3")
    assert "BJ(CI)" in b.workload(512, "bj", 4)
    assert "M = I" in b.workload(512, "none", 0)


def test_algorithmic_bytes_and_flops():
    b = load_bench()
    assert b.ALG_BYTES_PER_PT == 200.0            # 120 + 48 + 32
    assert b.ALG_BYTES_NONE == 168.0              # 24 + 24 + 24 + 64 + 32
    # 12 + 16 + 15 + 15 flops for the 4 sweeps + 4 for the fused p update
    assert b.FLOPS_PER_PT["fused_p_cheb"](4) == 62


def test_peaks_source_is_reported():
    b = load_bench()
    peak, src = b.peaks()
    assert peak > 1000.0 and isinstance(src, str) and src


def test_max_over_ranks_single_process_is_identity():
    b = load_bench()
    assert b.max_over_ranks(3.5) == 3.5


def test_reference_arm_samples_the_full_grid_for_driver_runs():
    """The driver's --steps 20 --warmup 5 run times the oracle on the same 512^3 workload as
    our arm; only longer runs fall back to a slab (bounded wall time)."""
    b = load_bench()
    assert b.reference_sample_planes(512, 20, 5) == 512
    ls = b.reference_sample_planes(512, 200, 10)
    assert 8 <= ls < 512 and ls % 8 == 0
