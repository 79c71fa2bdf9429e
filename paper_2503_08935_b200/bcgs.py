"""Thin ctypes binding of include/bcgs.h (libbcgs.so).  Argument marshalling only.

PyTorch supplies the device workspace, the caller's stream and (multi-rank) the process
group used to broadcast the NCCL unique id.  Every step of the solver runs in the CUDA
library; there is no CPU fallback: if the library cannot be loaded or no GPU is present,
`Solver` raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# BCGS_LIB: load another build of the same library (A/B timing of kernel changes)
LIB_PATH = os.environ.get("BCGS_LIB") or os.path.join(_PKG, "lib", "libbcgs.so")

OK, E_INVALID, E_CONFIG, E_SPECTRUM, E_CUDA, E_NCCL, NOT_CONVERGED, BREAKDOWN, E_STATE, E_COMM = range(10)
STATUS_NAMES = {0: "ok", 1: "invalid", 2: "config", 3: "spectrum", 4: "cuda", 5: "nccl",
                6: "not_converged", 7: "breakdown", 8: "state", 9: "comm"}
PC = {"none": 0, "gnocomm": 1, "bj": 2, "g": 3, "bj_bicgs": 4, "g_bicgs": 5}
MEM_DEVICE, MEM_HOST = 0, 1
OPT_KERNELS, OPT_GRAPH, OPT_PROFILE, OPT_POLL, OPT_TB_VARIANT = 0, 1, 2, 3, 4
OPT_MULTIPASS, OPT_ABLATE, OPT_SYNC2, OPT_EXACT_DOT, OPT_COMM_TIMEOUT = 8, 9, 10, 11, 12
OPT_PIPELINED, OPT_STENCIL, OPT_TB_SCHEDULE, OPT_PDL = 13, 14, 15, 16
HIST_CAP = 16384
MAX_DEGREE = 64

# Every symbol include/bcgs.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "bcgs_abi_version", "bcgs_status_string", "bcgs_workspace_bytes",
    "bcgs_chebyshev_constants", "bcgs_nccl_unique_id", "bcgs_create", "bcgs_create_local",
    "bcgs_destroy",
    "bcgs_last_error", "bcgs_set_option", "bcgs_set_rhs_random", "bcgs_set_rhs",
    "bcgs_set_boundary_value", "bcgs_set_initial_guess", "bcgs_set_preconditioner",
    "bcgs_set_eigen_bounds", "bcgs_solve", "bcgs_begin", "bcgs_iterate", "bcgs_finish",
    "bcgs_join",
    "bcgs_residual_history", "bcgs_scalar_history", "bcgs_get_solution",
    "bcgs_apply_operator", "bcgs_apply_preconditioner", "bcgs_dot", "bcgs_kernel_times",
    "bcgs_kernel_times_reset", "bcgs_set_inner_solver", "bcgs_inner_iterations",
    "bcgs_exact_dots", "bcgs_certification_info", "bcgs_create_p2p", "bcgs_p2p_handle", "bcgs_p2p_connect",
    "bcgs_create_local_p2p", "bcgs_get_phase_times",
]


# SPEC S:382 phase keys, in bcgs_get_phase_times order
PHASE_KEYS = ("preconditioner", "halo_exchange", "allreduce", "stencil_kernels",
              "vector_kernels", "total")


class BcgsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class GridDesc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64 * 3), ("h", ctypes.c_double), ("bc", ctypes.c_int32 * 6)]


BC_DIRICHLET, BC_NEUMANN = 0, 1


class Report(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("iterations", ctypes.c_int32), ("degree_warning", ctypes.c_int32),
                ("rel_residual", ctypes.c_double), ("true_rel_residual", ctypes.c_double),
                ("seconds", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_} | {
            "status_name": STATUS_NAMES.get(self.status, str(self.status))}


_lib = None


def load() -> ctypes.CDLL:
    """Load libbcgs.so.  Raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; "
                           "g.build()'` (nvcc, sm_100a)")
    lib = ctypes.CDLL(LIB_PATH)
    P, i32, i64, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sig = {
        "bcgs_abi_version": (i32, []),
        "bcgs_status_string": (ctypes.c_char_p, [i32]),
        "bcgs_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(GridDesc), i32]),
        "bcgs_chebyshev_constants": (i32, [ctypes.POINTER(GridDesc), i32, i32, i32, f64, f64,
                                           P, P, P]),
        "bcgs_nccl_unique_id": (i32, [P]),
        "bcgs_create": (i32, [ctypes.POINTER(GridDesc), i32, i32, P, i32, P, ctypes.c_size_t,
                              P, ctypes.POINTER(P)]),
        "bcgs_create_local": (i32, [ctypes.POINTER(GridDesc), i32, i32, ctypes.POINTER(P),
                                    ctypes.c_size_t, P, ctypes.POINTER(P)]),
        "bcgs_destroy": (None, [P]),
        "bcgs_last_error": (ctypes.c_char_p, [P]),
        "bcgs_set_option": (i32, [P, i32, i64]),
        "bcgs_set_rhs_random": (i32, [P, ctypes.c_uint64]),
        "bcgs_set_rhs": (i32, [P, P, i32]),
        "bcgs_set_boundary_value": (i32, [P, i32, f64]),
        "bcgs_set_initial_guess": (i32, [P, P, i32]),
        "bcgs_set_preconditioner": (i32, [P, i32, i32, f64, f64, i32]),
        "bcgs_set_eigen_bounds": (i32, [P, f64, f64]),
        "bcgs_solve": (i32, [P, f64, i32, i32, ctypes.POINTER(Report)]),
        "bcgs_begin": (i32, [P, f64, i32, i32]),
        "bcgs_iterate": (i32, [P, i32]),
        "bcgs_finish": (i32, [P, ctypes.POINTER(Report)]),
        "bcgs_join": (i32, [P]),
        "bcgs_residual_history": (i32, [P, P, i32]),
        "bcgs_scalar_history": (i32, [P, P, i32]),
        "bcgs_get_solution": (i32, [P, P, i32]),
        "bcgs_apply_operator": (i32, [P, P, P, i32]),
        "bcgs_apply_preconditioner": (i32, [P, P, P]),
        "bcgs_dot": (i32, [P, P, P, P]),
        "bcgs_kernel_times": (i32, [P, ctypes.c_char_p, i32, P, P, P, i32]),
        "bcgs_kernel_times_reset": (None, [P]),
        "bcgs_get_phase_times": (i32, [P, P]),
        "bcgs_set_inner_solver": (i32, [P, f64, i32]),
        "bcgs_inner_iterations": (i64, [P]),
        "bcgs_exact_dots": (ctypes.c_int32, [P]),
        "bcgs_certification_info": (i32, [P, P]),
        "bcgs_create_p2p": (i32, [P, i32, i32, i32, P, ctypes.c_size_t, P, P]),
        "bcgs_p2p_handle": (i32, [P, P]),
        "bcgs_p2p_connect": (i32, [P, P]),
        "bcgs_create_local_p2p": (i32, [P, i32, i32, P, ctypes.c_size_t, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def grid_desc(n, h: float, bc=None) -> GridDesc:
    """bc: six face kinds (x-, x+, y-, y+, z-, z+; 0 Dirichlet, 1 Neumann), default all 0."""
    n3 = (n, n, n) if np.isscalar(n) else tuple(n)
    g = GridDesc()
    g.n[0], g.n[1], g.n[2] = (int(v) for v in n3)
    g.h = float(h)
    for f, kind in enumerate(bc or (0,) * 6):
        g.bc[f] = int(kind)
    return g


def workspace_bytes(n, h: float, nranks: int = 1) -> int:
    return int(load().bcgs_workspace_bytes(ctypes.byref(grid_desc(n, h)), nranks))


def chebyshev_constants(n, h, nslab, pc, degree, c_min=10.0, c_max=1.0 - 1e-4, bc=None):
    ivl, cst, rho = np.zeros(2), np.zeros(7), np.zeros(max(degree, 1) + 1)
    st = load().bcgs_chebyshev_constants(ctypes.byref(grid_desc(n, h, bc)), nslab, PC[pc], degree,
                                         c_min, c_max, ivl.ctypes.data, cst.ctypes.data,
                                         rho.ctypes.data)
    if st:
        raise BcgsError(st, "bcgs_chebyshev_constants")
    return ivl, cst, rho


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = load().bcgs_nccl_unique_id(buf)
    if st:
        raise BcgsError(st, "bcgs_nccl_unique_id")
    return buf.raw


def _tensor_ptr(t):
    import torch
    assert t.dtype == torch.float64 and t.is_contiguous()
    return t.data_ptr(), (MEM_DEVICE if t.is_cuda else MEM_HOST)


class Solver:
    """One rank's context.  `n` = global unknowns (int or (nx, ny, nz)), `h` = spacing."""

    def __init__(self, n, h: float, *, rank: int = 0, nranks: int = 1,
                 nccl_id: bytes | None = None, device: int | None = None, stream=None,
                 bc=None, transport: str = "nccl", _ctx=None, _workspace=None):
        """transport (nranks > 1): "nccl" (nccl_id from rank 0) or "p2p" (peer memory:
        then every rank calls p2p_handle(), all-gathers the records and p2p_connect(...);
        see connect_p2p)."""
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("bcgs.Solver needs a CUDA device (no CPU fallback)")
        self.lib = load()
        self.n = (n, n, n) if np.isscalar(n) else tuple(int(v) for v in n)
        self.h = float(h)
        self.rank, self.nranks = rank, nranks
        self.device = torch.cuda.current_device() if device is None else device
        self.L = self.n[2] // nranks
        self.shape = (self.L, self.n[1], self.n[0])
        self.bc = tuple(bc) if bc is not None else (0,) * 6
        self.desc = grid_desc(self.n, h, self.bc)
        if _ctx is not None:                       # member of a local group
            self.ctx, self.workspace = _ctx, _workspace
            self.stream = stream
            return
        nbytes = self.lib.bcgs_workspace_bytes(ctypes.byref(self.desc), nranks)
        if nbytes == 0:
            raise BcgsError(E_CONFIG, f"grid {self.n} not divisible into {nranks} z-slabs")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{self.device}")
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        ctx = ctypes.c_void_p()
        if transport == "p2p" and nranks > 1:
            st = self.lib.bcgs_create_p2p(ctypes.byref(self.desc), rank, nranks, self.device,
                                          self.workspace.data_ptr(), nbytes,
                                          self.stream.cuda_stream, ctypes.byref(ctx))
        else:
            idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
            st = self.lib.bcgs_create(ctypes.byref(self.desc), rank, nranks, idbuf, self.device,
                                      self.workspace.data_ptr(), nbytes, self.stream.cuda_stream,
                                      ctypes.byref(ctx))
        self.ctx = ctx
        self._check(st, "bcgs_create")

    # ------------------------------------------------------------------ p2p transport
    def p2p_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(128)
        self._check(self.lib.bcgs_p2p_handle(self.ctx, buf), "bcgs_p2p_handle")
        return buf.raw

    def p2p_connect(self, handles: list[bytes]):
        blob = b"".join(handles)
        assert len(blob) == 128 * self.nranks
        buf = ctypes.create_string_buffer(blob, len(blob))
        self._check(self.lib.bcgs_p2p_connect(self.ctx, buf), "bcgs_p2p_connect")

    # ------------------------------------------------------------------ plumbing
    def _check(self, st, what):
        if st not in (OK,):
            msg = self.lib.bcgs_last_error(self.ctx) if self.ctx else b""
            raise BcgsError(st, f"{what}: {msg.decode() if msg else ''}")

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.bcgs_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, opt: int, value: int):
        self._check(self.lib.bcgs_set_option(self.ctx, opt, int(value)), "bcgs_set_option")

    # ------------------------------------------------------------------ inputs
    def set_rhs_random(self, seed: int):
        self._check(self.lib.bcgs_set_rhs_random(self.ctx, seed), "bcgs_set_rhs_random")

    def set_rhs(self, f):
        import torch
        if isinstance(f, np.ndarray):
            f = torch.from_numpy(np.ascontiguousarray(f, np.float64))
        assert tuple(f.shape) == self.shape or f.numel() == np.prod(self.shape)
        p, mem = _tensor_ptr(f)
        self._check(self.lib.bcgs_set_rhs(self.ctx, p, mem), "bcgs_set_rhs")

    def set_boundary_value(self, face: int, value: float):
        self._check(self.lib.bcgs_set_boundary_value(self.ctx, face, value),
                    "bcgs_set_boundary_value")

    def set_initial_guess(self, x0=None):
        import torch
        if x0 is None:
            self._check(self.lib.bcgs_set_initial_guess(self.ctx, None, 0), "x0")
            return
        if isinstance(x0, np.ndarray):
            x0 = torch.from_numpy(np.ascontiguousarray(x0, np.float64))
        p, mem = _tensor_ptr(x0)
        self._check(self.lib.bcgs_set_initial_guess(self.ctx, p, mem), "bcgs_set_initial_guess")

    def set_preconditioner(self, pc: str = "gnocomm", degree: int = 4, c_min: float = 10.0,
                           c_max: float = 1.0 - 1e-4, blocks_per_rank: int = 1):
        self._check(self.lib.bcgs_set_preconditioner(self.ctx, PC[pc], degree, c_min, c_max,
                                                     blocks_per_rank),
                    "bcgs_set_preconditioner")

    def set_inner_solver(self, tol: float, max_iter: int = 500):
        """BJ(BiCGS) / G(BiCGS): inner relative tolerance and iteration cap."""
        self._check(self.lib.bcgs_set_inner_solver(self.ctx, tol, max_iter),
                    "bcgs_set_inner_solver")

    def inner_iterations(self) -> int:
        return int(self.lib.bcgs_inner_iterations(self.ctx))

    def exact_dots(self) -> int:
        """Dots recomputed on the exact path since the last begin (R19)."""
        return int(self.lib.bcgs_exact_dots(self.ctx))

    def certification_info(self) -> dict:
        out = np.zeros(10)
        self._check(self.lib.bcgs_certification_info(self.ctx, out.ctypes.data),
                    "bcgs_certification_info")
        keys = ["stage", "dot", "D", "r", "e", "E", "gap_up", "gap_down", "sum_abs", "refused"]
        return dict(zip(keys, map(float, out)))

    def set_eigen_bounds(self, a: float, b: float):
        self._check(self.lib.bcgs_set_eigen_bounds(self.ctx, a, b), "bcgs_set_eigen_bounds")

    # ------------------------------------------------------------------ solve
    def solve(self, tol: float = 1e-8, max_iter: int = 5000, fixed_iters: int = 0) -> dict:
        rep = Report()
        st = self.lib.bcgs_solve(self.ctx, tol, max_iter, fixed_iters, ctypes.byref(rep))
        if st not in (OK, NOT_CONVERGED, BREAKDOWN):
            self._check(st, "bcgs_solve")
        return rep.as_dict()

    def begin(self, tol: float = 1e-8, max_iter: int = 5000, fixed_iters: int = 0):
        self._check(self.lib.bcgs_begin(self.ctx, tol, max_iter, fixed_iters), "bcgs_begin")

    def iterate(self, n: int):
        self._check(self.lib.bcgs_iterate(self.ctx, n), "bcgs_iterate")

    def join_stream(self):
        """Make the caller's stream wait for the library stream (stream-ordered, no host sync)."""
        self._check(self.lib.bcgs_join(self.ctx), "bcgs_join")

    def finish(self) -> dict:
        rep = Report()
        st = self.lib.bcgs_finish(self.ctx, ctypes.byref(rep))
        if st not in (OK, NOT_CONVERGED, BREAKDOWN):
            self._check(st, "bcgs_finish")
        return rep.as_dict()

    def residual_history(self) -> np.ndarray:
        buf = np.zeros(HIST_CAP + 1)
        m = self.lib.bcgs_residual_history(self.ctx, buf.ctypes.data, HIST_CAP + 1)
        return buf[:m].copy()

    def scalar_history(self) -> np.ndarray:
        buf = np.zeros((HIST_CAP, 8))
        m = self.lib.bcgs_scalar_history(self.ctx, buf.ctypes.data, HIST_CAP)
        return buf[:m].copy()

    def solution(self, device: bool = True):
        import torch
        if device:
            x = torch.empty(self.shape, dtype=torch.float64, device=f"cuda:{self.device}")
        else:
            x = torch.empty(self.shape, dtype=torch.float64).pin_memory()
        p, mem = _tensor_ptr(x)
        self._check(self.lib.bcgs_get_solution(self.ctx, p, mem), "bcgs_get_solution")
        return x

    # ------------------------------------------------------------------ single steps
    def apply_operator(self, v, block_local: bool = False):
        import torch
        out = torch.empty_like(v)
        self._check(self.lib.bcgs_apply_operator(self.ctx, v.data_ptr(), out.data_ptr(),
                                                 int(block_local)), "bcgs_apply_operator")
        return out

    def apply_preconditioner(self, v):
        import torch
        out = torch.empty_like(v)
        self._check(self.lib.bcgs_apply_preconditioner(self.ctx, v.data_ptr(), out.data_ptr()),
                    "bcgs_apply_preconditioner")
        return out

    def dot(self, a, b) -> float:
        r = ctypes.c_double(0.0)
        self._check(self.lib.bcgs_dot(self.ctx, a.data_ptr(), b.data_ptr(), ctypes.byref(r)),
                    "bcgs_dot")
        return r.value

    def kernel_times(self) -> dict:
        names = ctypes.create_string_buffer(4096)
        ms = np.zeros(64)
        calls = np.zeros(64, np.int64)
        byts = np.zeros(64)
        m = self.lib.bcgs_kernel_times(self.ctx, names, 4096, ms.ctypes.data, calls.ctypes.data,
                                       byts.ctypes.data, 64)
        keys = names.value.decode().split("\n")[:m]
        return {k: {"ms": float(ms[i]), "calls": int(calls[i]), "bytes_per_call": float(byts[i])}
                for i, k in enumerate(keys) if calls[i] > 0}

    def kernel_times_reset(self):
        self.lib.bcgs_kernel_times_reset(self.ctx)

    def phase_times(self) -> dict:
        """Milliseconds per SPEC phase key accumulated while OPT_PROFILE = 1."""
        out = np.zeros(6)
        self._check(self.lib.bcgs_get_phase_times(self.ctx, out.ctypes.data),
                    "bcgs_get_phase_times")
        return dict(zip(PHASE_KEYS, (float(v) for v in out)))


def connect_p2p(solver: "Solver", group=None):
    """All-gather the ranks' p2p records through torch.distributed (any backend) and connect."""
    import torch.distributed as dist
    recs = [None] * solver.nranks
    dist.all_gather_object(recs, solver.p2p_handle(), group=group)
    solver.p2p_connect(recs)


def local_group(n, h: float, nranks: int, device: int | None = None, bc=None,
                transport: str = "copy") -> list:
    """nranks Solver contexts on ONE GPU (drive each from its own thread).  transport
    "copy": halos / reductions by stream-ordered device copies + a host barrier (the NCCL
    path's sequence, bcgs_create_local); "p2p": the peer-memory kernels of p2p.cuh with
    direct pointers (bcgs_create_local_p2p)."""
    import torch
    lib = load()
    device = torch.cuda.current_device() if device is None else device
    desc = grid_desc(n, h, bc)
    nbytes = lib.bcgs_workspace_bytes(ctypes.byref(desc), nranks)
    if nbytes == 0:
        raise BcgsError(E_CONFIG, "grid not divisible into z-slabs")
    wss = [torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}") for _ in range(nranks)]
    ptrs = (ctypes.c_void_p * nranks)(*[w.data_ptr() for w in wss])
    outs = (ctypes.c_void_p * nranks)()
    stream = torch.cuda.current_stream(device)
    create = lib.bcgs_create_local_p2p if transport == "p2p" else lib.bcgs_create_local
    st = create(ctypes.byref(desc), nranks, device, ptrs, nbytes, stream.cuda_stream, outs)
    if st:
        raise BcgsError(st, "bcgs_create_local")
    return [Solver(n, h, rank=r, nranks=nranks, device=device, stream=stream, bc=bc,
                   _ctx=ctypes.c_void_p(outs[r]), _workspace=wss[r]) for r in range(nranks)]
