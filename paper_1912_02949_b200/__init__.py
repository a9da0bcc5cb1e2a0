"""B200-native SketchyCGAL MaxCut hot path (arXiv 1912.02949) -- Python binding.

Thin ctypes binding of the C ABI in ``include/sketchycgal.h``: argument
marshalling only.  Every step of the iteration runs in the CUDA kernels of
``csrc/`` (sm_100a); there is no CPU fallback -- ``load()`` raises if the
library is missing or no GPU is visible.  PyTorch is used only for device
selection / streams and ``torch.distributed`` plumbing (multi-GPU bootstrap).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(_HERE)
LIB_DIR = os.path.join(_HERE, "lib")
LIB_PATH = os.environ.get("SCG_LIB") or os.path.join(LIB_DIR, "libsketchycgal.so")
SOURCES = [os.path.join(_HERE, "csrc", f) for f in ("sketchycgal.cu", "kernels.cuh", "xsum.cuh")]
HEADERS = [os.path.join(ROOT, "include", "sketchycgal.h"), os.path.join(ROOT, "scg_inputs", "include", "scg_rng.h")]

SCG_SCALE = 1 << 0
SCG_TRACE_CORRECT = 1 << 1
SCG_REGENERATE = 1 << 2
SCG_TRACE_LE = 1 << 3
SCG_INEQ = 1 << 4
SCG_PROFILE = 1 << 8
SCG_NO_PDL = 1 << 9
SCG_FUSED_PASS1 = 1 << 10
SCG_WS_SPMV = 1 << 11
SCG_TMA_B = 1 << 12
SCG_DEBUG_LOG = 1 << 13
SCG_NO_ELL = 1 << 14
SCG_FUSED_RNG = 1 << 15
SCG_NO_RESIDENT = 1 << 17
SCG_SERIAL_RNG = 1 << 18
SCG_INLINE_PULL = 1 << 19

STATUS = {0: "SCG_OK", -1: "SCG_EINVAL", -2: "SCG_ENOMEM", -3: "SCG_ECUDA", -4: "SCG_ENCCL", -5: "SCG_ECHOL",
          -6: "SCG_ESTATE", -7: "SCG_ERANGE", -8: "SCG_EUNSUPPORTED", -9: "SCG_ECOMM"}


def _nccl_paths():
    try:
        import nvidia.nccl as nn
        base = os.path.dirname(nn.__file__) if getattr(nn, "__file__", None) else list(nn.__path__)[0]
    except Exception:
        base = os.path.join(sys.prefix, "lib", f"python{sys.version_info.major}.{sys.version_info.minor}",
                            "site-packages", "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
        return inc, lib
    return None, None


def nvcc_cmd(out: str, defines=()) -> list[str]:
    cmd = ["nvcc", *[f"-D{d}" for d in defines], "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false",
           "-std=c++17", "-Xcompiler", "-fPIC,-fopenmp", "-shared", "-cudart", "static", "-lgomp",
           os.path.join(_HERE, "csrc", "sketchycgal.cu"), "-o", out]
    inc, lib = _nccl_paths()
    if inc:
        cmd[1:1] = ["-DSCG_WITH_NCCL", f"-I{inc}"]
        cmd += [f"-L{lib}", "-l:libnccl.so.2", f"-Xlinker=-rpath={lib}"]
    return cmd


def build(force: bool = False) -> str:
    """Compile the CUDA library for sm_100a in-tree (nvcc cross-compiles without a GPU)."""
    os.makedirs(LIB_DIR, exist_ok=True)
    newest = max(os.path.getmtime(p) for p in SOURCES + HEADERS)
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= newest:
        return LIB_PATH
    tmp = LIB_PATH + f".tmp{os.getpid()}"
    subprocess.check_call(nvcc_cmd(tmp))
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


class IterRec(ctypes.Structure):
    _fields_ = [("t", ctypes.c_int64), ("q", ctypes.c_int32), ("k", ctypes.c_int32), ("theta", ctypes.c_double),
                ("xi", ctypes.c_double), ("c", ctypes.c_double), ("p", ctypes.c_double),
                ("znorm", ctypes.c_double), ("gamma", ctypes.c_double), ("tau", ctypes.c_double),
                ("gap", ctypes.c_double), ("bound", ctypes.c_double)]


class KStat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_int64), ("total_ms", ctypes.c_double),
                ("bytes_per_launch", ctypes.c_double)]


class Csr(ctypes.Structure):
    _fields_ = [("n_global", ctypes.c_int64), ("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64),
                ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p), ("val", ctypes.c_void_p),
                ("has_diagonal", ctypes.c_int32)]


ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int64)
BARRIER_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p)


class HostCommStruct(ctypes.Structure):
    _fields_ = [("ctx", ctypes.c_void_p), ("allgather", ALLGATHER_FN), ("allreduce_sum", ALLREDUCE_FN),
                ("barrier", BARRIER_FN), ("sync_collectives", ctypes.c_int32)]


class Dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("nccl_unique_id", ctypes.c_void_p),
                ("row_splits", ctypes.c_void_p), ("emulate", ctypes.c_int32),
                ("host_comm", ctypes.POINTER(HostCommStruct))]


class TorchHostComm:
    """scg_host_comm over torch.distributed (any backend with CPU tensors, e.g. gloo): the setup and
    one-shot exchanges of a multi-process run without NCCL.  ``sync_collectives=True`` makes every
    device collective meet on the host first (ranks may then share one GPU: no kernel ever waits for
    another rank's kernel) -- include/sketchycgal.h."""

    def __init__(self, group=None, sync_collectives: bool = True):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)

        def allgather(ctx, src, dst, nbytes):
            try:
                import torch
                t = torch.frombuffer(bytearray(ctypes.string_at(src, nbytes)), dtype=torch.uint8)
                out = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(self.world)]
                dist.all_gather(out, t, group=self.group)
                buf = b"".join(o.numpy().tobytes() for o in out)
                ctypes.memmove(dst, buf, len(buf))
                return 0
            except Exception:
                return -1

        def allreduce_sum(ctx, buf, count):
            try:
                import torch
                a = np.ctypeslib.as_array(buf, shape=(count,))
                t = torch.from_numpy(a.copy())
                dist.all_reduce(t, group=self.group)
                a[:] = t.numpy()
                return 0
            except Exception:
                return -1

        def barrier(ctx):
            try:
                dist.barrier(group=self.group)
                return 0
            except Exception:
                return -1

        self._fns = (ALLGATHER_FN(allgather), ALLREDUCE_FN(allreduce_sum), BARRIER_FN(barrier))
        self.struct = HostCommStruct(None, *self._fns, 1 if sync_collectives else 0)


EXPORTS = ["sketchycgal_maxcut_init", "sketchycgal_step", "sketchycgal_synchronize", "sketchycgal_reconstruct",
           "sketchycgal_objective", "sketchycgal_feasibility", "sketchycgal_round", "sketchycgal_iter_log",
           "sketchycgal_get_state", "sketchycgal_apply_D", "sketchycgal_iterations", "sketchycgal_launch_count",
           "sketchycgal_kernel_stats", "sketchycgal_reset_stats", "sketchycgal_nccl_unique_id",
           "sketchycgal_row_splits", "sketchycgal_halo_plan", "sketchycgal_run",
           "sketchycgal_selftest_division", "sketchycgal_selftest_xsum", "sketchycgal_last_error", "sketchycgal_destroy",
           "sketchycgal_maxcut_alpha_doubling", "sketchycgal_set_box", "sketchycgal_set_ball", "sketchycgal_set_ball_l1",
           "sketchycgal_set_lanczos_q"]

_lib = None


def open_library(path: str = LIB_PATH):
    """dlopen the library and declare the ABI (no GPU needed)."""
    lib = ctypes.CDLL(path)
    P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    lib.sketchycgal_maxcut_init.restype = ctypes.c_int
    lib.sketchycgal_maxcut_init.argtypes = [ctypes.POINTER(P), ctypes.POINTER(Csr), I32, D, D, ctypes.c_uint64,
                                            ctypes.c_uint32, ctypes.POINTER(Dist), I32, P]
    for name, args in [("sketchycgal_step", [P, I64]), ("sketchycgal_synchronize", [P]),
                       ("sketchycgal_reconstruct", [P, P, P, P]), ("sketchycgal_objective", [P, P]),
                       ("sketchycgal_feasibility", [P, P]), ("sketchycgal_round", [P, P, P]),
                       ("sketchycgal_iter_log", [P, I64, I64, P]), ("sketchycgal_get_state", [P, I32, P]),
                       ("sketchycgal_apply_D", [P, P, P]), ("sketchycgal_nccl_unique_id", [P])]:
        getattr(lib, name).restype = ctypes.c_int
        getattr(lib, name).argtypes = args
    lib.sketchycgal_iterations.restype = I64
    lib.sketchycgal_iterations.argtypes = [P]
    lib.sketchycgal_launch_count.restype = I64
    lib.sketchycgal_launch_count.argtypes = [P]
    lib.sketchycgal_kernel_stats.restype = I32
    lib.sketchycgal_kernel_stats.argtypes = [P, P, I32]
    lib.sketchycgal_reset_stats.restype = None
    lib.sketchycgal_reset_stats.argtypes = [P]
    lib.sketchycgal_run.restype = ctypes.c_int
    lib.sketchycgal_run.argtypes = [P, I64, D, I64, ctypes.POINTER(I64)]
    lib.sketchycgal_set_lanczos_q.restype = ctypes.c_int
    lib.sketchycgal_set_lanczos_q.argtypes = [P, I32]
    lib.sketchycgal_set_box.restype = ctypes.c_int
    lib.sketchycgal_set_box.argtypes = [P, D, D]
    lib.sketchycgal_set_ball.restype = ctypes.c_int
    lib.sketchycgal_set_ball.argtypes = [P, D]
    lib.sketchycgal_set_ball_l1.restype = ctypes.c_int
    lib.sketchycgal_set_ball_l1.argtypes = [P, D]
    lib.sketchycgal_maxcut_alpha_doubling.restype = ctypes.c_int
    lib.sketchycgal_maxcut_alpha_doubling.argtypes = [ctypes.POINTER(P), ctypes.POINTER(Csr), I32, D, D,
                                                      ctypes.c_uint64, ctypes.c_uint32, I32, P, I64, D, I32, P, P,
                                                      ctypes.POINTER(I32), ctypes.POINTER(I32)]
    lib.sketchycgal_row_splits.restype = ctypes.c_int
    lib.sketchycgal_row_splits.argtypes = [P, I64, I32, P]
    lib.sketchycgal_halo_plan.restype = I64
    lib.sketchycgal_halo_plan.argtypes = [P, P, I64, I64, P, I32, P]
    lib.sketchycgal_selftest_division.restype = ctypes.c_int
    lib.sketchycgal_selftest_division.argtypes = [I32, I64, ctypes.c_uint64, ctypes.POINTER(I64)]
    lib.sketchycgal_selftest_xsum.restype = ctypes.c_int
    lib.sketchycgal_selftest_xsum.argtypes = [I32, P, I64, I32, I32, ctypes.POINTER(D), ctypes.POINTER(I32)]
    lib.sketchycgal_last_error.restype = ctypes.c_char_p
    lib.sketchycgal_last_error.argtypes = [P]
    lib.sketchycgal_destroy.restype = None
    lib.sketchycgal_destroy.argtypes = [P]
    return lib


def row_splits(row_ptr, world: int) -> np.ndarray:
    """Balanced contiguous row split (rows + nonzeros per rank) -- host code of the library, no GPU."""
    rp = _c64(row_ptr, np.int64)
    out = np.zeros(world + 1, dtype=np.int64)
    st = load().sketchycgal_row_splits(rp.ctypes.data, len(rp) - 1, int(world), out.ctypes.data)
    if st != 0:
        raise ScgError(f"sketchycgal_row_splits: {STATUS.get(st, st)}")
    return out


def halo_plan(row_ptr, col, row_begin: int, row_end: int, splits) -> tuple[np.ndarray, int]:
    """Reader-rank bitmask of each own row of a shard (library host code, no GPU).  row_ptr/col are the
    shard's own rows (row_ptr[0] may be nonzero)."""
    rp = _c64(row_ptr, np.int64)
    cc = _c64(col, np.int32)
    sp = _c64(splits, np.int64)
    mask = np.zeros(max(1, row_end - row_begin), dtype=np.uint8)
    h = load().sketchycgal_halo_plan(rp.ctypes.data, cc.ctypes.data, int(row_begin), int(row_end), sp.ctypes.data,
                                     len(sp) - 1, mask.ctypes.data)
    if h < 0:
        raise ScgError("sketchycgal_halo_plan failed")
    return mask[:row_end - row_begin], int(h)


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = load().sketchycgal_nccl_unique_id(buf)
    if st != 0:
        raise ScgError(f"sketchycgal_nccl_unique_id: {STATUS.get(st, st)}")
    return buf.raw


def load():
    """Load the CUDA library.  Fails loudly (no fallback) without the library or a GPU."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA library {LIB_PATH} is missing: run __graft_entry__.build()")
        _lib = open_library(LIB_PATH)
    return _lib


class ScgError(RuntimeError):
    pass


def selftest_division(n: int = 1 << 26, seed: int = 1, device: int = 0) -> int:
    """Mismatches of the kernels' shared-divisor division vs IEEE division on n random pairs."""
    out = ctypes.c_int64(-1)
    st = load().sketchycgal_selftest_division(int(device), int(n), int(seed), ctypes.byref(out))
    if st != 0:
        raise ScgError(f"selftest: {STATUS.get(st, st)}")
    return int(out.value)


def selftest_xsum(values, grid: int = 64, block: int = 256, device: int = 0):
    """(xsum(values) rounded once, range error flag) from the device's per-thread exact accumulators."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    out, rerr = ctypes.c_double(0.0), ctypes.c_int32(0)
    st = load().sketchycgal_selftest_xsum(int(device), v.ctypes.data, int(v.size), int(grid), int(block),
                                          ctypes.byref(out), ctypes.byref(rerr))
    if st != 0:
        raise ScgError(f"selftest_xsum: {STATUS.get(st, st)}")
    return float(out.value), int(rerr.value)


def _c64(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class SketchyCGAL:
    """SketchyCGAL MaxCut solver context (sketchycgal_maxcut_init ... destroy).

    One GPU by default.  ``shards=P`` runs the row-sharded path with P emulated ranks
    inside this one context on one device (all per-row outputs still cover all n rows).
    Multi-process (one process per GPU): pass ``rank``, ``world``, ``splits`` (world+1
    row offsets) and ``nccl_id`` (the 128 bytes of ``nccl_unique_id()`` from rank 0);
    ``L`` may be the full CSR, the rank's rows are taken from it.

    Execution options (bitwise-neutral): ``pdl`` (programmatic dependent
    launches, default on), ``fused_pass1`` (persistent pass-1 kernel), ``ws_spmv``
    (warp-specialized TMA SpMV), ``tma_b`` (TMA-staged recurrence kernel), ``ell`` (ELL-W layout when
    every row has <= 8 entries, default on), ``debug_log``.
    """

    def __init__(self, L, R: int, alpha: float | None = None, beta0: float = 1.0, seed: int = 0,
                 scale: bool = True, trace_correct: bool = True, profile: bool = False, device: int = 0,
                 stream=None, regenerate: bool = False, trace_le: bool = False, shards: int = 1, splits=None,
                 rank: int = 0, world: int = 1, nccl_id: bytes | None = None, ineq: bool = False,
                 box: tuple | None = None, ball: float | None = None,
                 l1_ball: float | None = None, pdl: bool = True, fused_pass1: bool = False, ws_spmv: bool = False,
                 tma_b: bool = False, debug_log: bool = False, qfix: int = 0, ell: bool = True,
                 side_rng: bool = True, host_comm: "TorchHostComm | None" = None, resident: bool = True,
                 serial_rng: bool = False, inline_pull: bool = False):
        self.lib = load()
        self.n = int(L.n)
        self.R = int(R)
        dist = None
        self._splits = None
        if shards > 1 or world > 1:
            P = shards if shards > 1 else world
            sp = row_splits(L.row_ptr, P) if splits is None else _c64(splits, np.int64)
            self._splits = sp
            self._uid = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
            self._host_comm = host_comm  # keeps the callbacks alive for the context's lifetime
            dist = Dist(0 if shards > 1 else int(rank), int(P), ctypes.addressof(self._uid) if self._uid else None,
                        sp.ctypes.data, 1 if shards > 1 else 0,
                        ctypes.pointer(host_comm.struct) if (host_comm is not None and shards <= 1) else None)
        if world > 1 and shards <= 1:
            self.row_begin, self.row_end = int(self._splits[rank]), int(self._splits[rank + 1])
        else:
            self.row_begin, self.row_end = 0, self.n
        self.nl = self.row_end - self.row_begin
        rp = _c64(L.row_ptr, np.int64)
        col = _c64(L.col, np.int32)
        val = _c64(L.val, np.float64)
        if self.row_begin != 0 or self.row_end != self.n:  # local rows of a full CSR
            a, b = int(rp[self.row_begin]), int(rp[self.row_end])
            col, val = col[a:b], val[a:b]
            rp = rp[self.row_begin:self.row_end + 1] - a
        self._keep = (rp, col, val)
        csr = Csr(self.n, self.row_begin, self.row_end, rp.ctypes.data, col.ctypes.data, val.ctypes.data, 1)
        flags = (SCG_SCALE if scale else 0) | (SCG_TRACE_CORRECT if trace_correct else 0) | \
                (SCG_PROFILE if profile else 0) | (SCG_REGENERATE if regenerate else 0) | \
                (SCG_TRACE_LE if trace_le else 0) | (SCG_INEQ if ineq else 0) | (0 if pdl else SCG_NO_PDL) | \
                (SCG_FUSED_PASS1 if fused_pass1 else 0) | (SCG_WS_SPMV if ws_spmv else 0) | \
                (SCG_TMA_B if tma_b else 0) | (SCG_DEBUG_LOG if debug_log else 0) | (0 if ell else SCG_NO_ELL) | \
                (0 if side_rng else SCG_FUSED_RNG) | (0 if resident else SCG_NO_RESIDENT) | \
                (SCG_SERIAL_RNG if serial_rng else 0) | (SCG_INLINE_PULL if inline_pull else 0)
        self._h = ctypes.c_void_p()
        dptr = None
        if dist is not None:
            self._dist = dist
            dptr = ctypes.byref(dist)
        st = self.lib.sketchycgal_maxcut_init(ctypes.byref(self._h), ctypes.byref(csr), self.R,
                                              float(self.n if alpha is None else alpha), float(beta0), int(seed),
                                              flags, dptr, int(device), stream)
        if st != 0:
            raise ScgError(f"sketchycgal_maxcut_init: {STATUS.get(st, st)}")
        if qfix:  # fixed Lanczos bound (Alg. 2 input q) instead of the q_t schedule
            self._check(self.lib.sketchycgal_set_lanczos_q(self._h, int(qfix)), "sketchycgal_set_lanczos_q")
        if box is not None:  # K = {lo <= u <= hi}
            self._check(self.lib.sketchycgal_set_box(self._h, float(box[0]), float(box[1])), "sketchycgal_set_box")
        if ball is not None:  # K = {||u - 1|| <= delta} (reading R34)
            self._check(self.lib.sketchycgal_set_ball(self._h, float(ball)), "sketchycgal_set_ball")
        if l1_ball is not None:  # K = {||u - 1||_1 <= delta} (reading R35)
            self._check(self.lib.sketchycgal_set_ball_l1(self._h, float(l1_ball)), "sketchycgal_set_ball_l1")

    @classmethod
    def alpha_doubling(cls, L, R: int, alpha0: float, T: int, rtol: float = 1e-2, max_rounds: int = 8,
                       beta0: float = 1.0, seed: int = 0, scale: bool = True, trace_correct: bool = True,
                       device: int = 0, stream=None):
        """Standard-form driver through ``sketchycgal_maxcut_alpha_doubling``:
        trace-bounded solves tr X <= alpha_i, alpha_{i+1} = 2 alpha_i, until the implicit objective
        repeats within ``rtol``.  Returns (context of the last round, alphas, objectives, converged)."""
        self = cls.__new__(cls)
        self.lib = load()
        self.n, self.R = int(L.n), int(R)
        self._splits = None
        self.row_begin, self.row_end, self.nl = 0, self.n, self.n
        rp, col, val = _c64(L.row_ptr, np.int64), _c64(L.col, np.int32), _c64(L.val, np.float64)
        self._keep = (rp, col, val)
        csr = Csr(self.n, 0, self.n, rp.ctypes.data, col.ctypes.data, val.ctypes.data, 1)
        flags = (SCG_SCALE if scale else 0) | (SCG_TRACE_CORRECT if trace_correct else 0)
        alphas = np.zeros(int(max_rounds))
        objs = np.zeros(int(max_rounds))
        rounds, conv = ctypes.c_int32(0), ctypes.c_int32(0)
        self._h = ctypes.c_void_p()
        st = self.lib.sketchycgal_maxcut_alpha_doubling(
            ctypes.byref(self._h), ctypes.byref(csr), self.R, float(alpha0), float(beta0), int(seed), flags,
            int(device), stream, int(T), float(rtol), int(max_rounds), alphas.ctypes.data, objs.ctypes.data,
            ctypes.byref(rounds), ctypes.byref(conv))
        if st != 0:
            raise ScgError(f"sketchycgal_maxcut_alpha_doubling: {STATUS.get(st, st)}")
        k = rounds.value
        return self, alphas[:k].copy(), objs[:k].copy(), bool(conv.value)

    def _check(self, st, what):
        if st != 0:
            msg = self.lib.sketchycgal_last_error(self._h)
            raise ScgError(f"{what}: {STATUS.get(st, st)} {msg.decode() if msg else ''}")

    def close(self):
        if getattr(self, "_h", None):
            self.lib.sketchycgal_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, T: int):
        self._check(self.lib.sketchycgal_step(self._h, int(T)), "sketchycgal_step")

    def run(self, T_max: int, eps: float = 0.1, check_every: int = 64):
        """Iterate until the stopping rule holds or T_max more iterations ran;
        returns the first iteration t meeting it, or None."""
        out = ctypes.c_int64(-1)
        self._check(self.lib.sketchycgal_run(self._h, int(T_max), float(eps), int(check_every), ctypes.byref(out)),
                    "sketchycgal_run")
        return None if out.value < 0 else int(out.value)

    def synchronize(self):
        self._check(self.lib.sketchycgal_synchronize(self._h), "sketchycgal_synchronize")

    @property
    def t(self) -> int:
        return int(self.lib.sketchycgal_iterations(self._h))

    @property
    def launches(self) -> int:
        return int(self.lib.sketchycgal_launch_count(self._h))

    def iter_log(self, t0: int = 1, count: int | None = None) -> np.ndarray:
        count = self.t - t0 + 1 if count is None else count
        buf = (IterRec * count)()
        self._check(self.lib.sketchycgal_iter_log(self._h, int(t0), int(count), buf), "sketchycgal_iter_log")
        return np.array([(r.t, r.q, r.k, r.theta, r.xi, r.c, r.p, r.znorm, r.gamma, r.tau, r.gap, r.bound)
                         for r in buf], dtype=np.float64).reshape(count, 12)

    def state(self, which: str) -> np.ndarray:
        idx = {"z": 0, "y": 1, "S": 2, "Omega": 3, "v": 4, "d": 5, "cdiag": 6}[which]
        size = self.nl * (self.R if which in ("S", "Omega") else 1)
        out = np.empty(size, dtype=np.float64)
        self._check(self.lib.sketchycgal_get_state(self._h, idx, out.ctypes.data), "sketchycgal_get_state")
        return out.reshape(self.R, self.nl).T if which in ("S", "Omega") else out

    def apply_D(self, x) -> np.ndarray:
        x = _c64(x, np.float64)
        y = np.empty(self.nl, dtype=np.float64)
        self._check(self.lib.sketchycgal_apply_D(self._h, x.ctypes.data, y.ctypes.data), "sketchycgal_apply_D")
        return y

    def reconstruct(self, want_U: bool = True):
        U = np.empty((self.R, self.nl), dtype=np.float64) if want_U else None
        lam = np.empty(self.R, dtype=np.float64)
        err = np.empty(self.R, dtype=np.float64)
        self._check(self.lib.sketchycgal_reconstruct(self._h, U.ctypes.data if want_U else None, lam.ctypes.data,
                                                     err.ctypes.data), "sketchycgal_reconstruct")
        return (U.T if want_U else None), lam, err

    def objective(self):
        out = np.empty(2, dtype=np.float64)
        self._check(self.lib.sketchycgal_objective(self._h, out.ctypes.data), "sketchycgal_objective")
        return out

    def feasibility(self):
        out = np.empty(3, dtype=np.float64)
        self._check(self.lib.sketchycgal_feasibility(self._h, out.ctypes.data), "sketchycgal_feasibility")
        return out

    def round(self):
        chi = np.empty(self.nl, dtype=np.int8)
        w = ctypes.c_double()
        self._check(self.lib.sketchycgal_round(self._h, chi.ctypes.data, ctypes.byref(w)), "sketchycgal_round")
        return chi, w.value

    def kernel_stats(self):
        buf = (KStat * 24)()
        n = self.lib.sketchycgal_kernel_stats(self._h, buf, 24)
        return [dict(name=buf[i].name.decode(), launches=buf[i].launches, total_ms=buf[i].total_ms,
                     bytes_per_launch=buf[i].bytes_per_launch) for i in range(max(n, 0))]

    def reset_stats(self):
        self.lib.sketchycgal_reset_stats(self._h)
