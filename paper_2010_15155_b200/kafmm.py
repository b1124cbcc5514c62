"""ctypes binding of libkafmm.so (include/kafmm.h).  Argument marshalling only.

PyTorch is used for device memory and streams: tensors are passed to the C
ABI as raw pointers (``Tensor.data_ptr()``).  Every step of the evaluation
runs in the library's CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
KERNELS = {"laplace_pgrad": 1, "stokeslet": 2, "rpy": 3, "stokes_reg_vel": 4, "stokes_reg_vel_omega": 5,
           "laplace_pgradgrad": 6, "laplace_qpgradgrad": 7}
N_STAGES = 13


class KafmmError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: status {status} ({detail})")
        self.status = status


class Info(C.Structure):
    _fields_ = [("n_points", C.c_int64), ("kernel", C.c_int), ("p", C.c_int), ("max_pts", C.c_int),
                ("depth", C.c_int), ("k_s", C.c_int), ("k_t", C.c_int), ("n_surf", C.c_int),
                ("n_equiv", C.c_int), ("kept_up", C.c_int), ("kept_dn", C.c_int),
                ("n_boxes", C.c_int64), ("n_leaves", C.c_int64), ("n_u_pairs", C.c_int64),
                ("n_v_pairs", C.c_int64), ("n_w_pairs", C.c_int64), ("n_p2p", C.c_int64),
                ("workspace_bytes", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def lib_path() -> str:
    return os.environ.get("KAFMM_LIB", os.path.join(HERE, "libkafmm.so"))


_LIB = None

# (name, restype, argtypes)
_SIGS = [
    ("kafmm_kernel_dims", C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("kafmm_setup", C.c_int, [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    ("kafmm_set_stream", C.c_int, [C.c_void_p, C.c_void_p]),
    ("kafmm_eval", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("kafmm_eval_host", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("kafmm_check_values", C.c_int, [C.c_void_p, C.c_void_p]),
    ("kafmm_sync", C.c_int, [C.c_void_p]),
    ("kafmm_destroy", None, [C.c_void_p]),
    ("kafmm_status_string", C.c_char_p, [C.c_int]),
    ("kafmm_last_error", C.c_char_p, []),
    ("kafmm_get_info", C.c_int, [C.c_void_p, C.POINTER(Info)]),
    ("kafmm_get_tree", C.c_int, [C.c_void_p] + [C.c_void_p] * 6),
    ("kafmm_get_permutation", C.c_int, [C.c_void_p, C.c_void_p]),
    ("kafmm_get_list", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    ("kafmm_set_timing", C.c_int, [C.c_void_p, C.c_int]),
    ("kafmm_stage_times", C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
    ("kafmm_stage_name", C.c_char_p, [C.c_int]),
    ("kafmm_launch_count", C.c_int, [C.c_void_p, C.POINTER(C.c_int)]),
    ("kafmm_fp64_peak", C.c_int, [C.c_int, C.POINTER(C.c_double)]),
    ("kafmm_set_m2l_mode", C.c_int, [C.c_void_p, C.c_int]),
    ("kafmm_get_m2l_mode", C.c_int, [C.c_void_p, C.POINTER(C.c_int)]),
    ("kafmm_fft_stats", C.c_int, [C.c_void_p, C.c_void_p]),
    ("kafmm_set_graph", C.c_int, [C.c_void_p, C.c_int]),
    ("kafmm_setup2", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int,
                               C.POINTER(C.c_void_p)]),
    ("kafmm_eval2", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("kafmm_get_unique_id", C.c_int, [C.c_void_p]),
    ("kafmm_setup_dist", C.c_int, [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                   C.POINTER(C.c_void_p)]),
    ("kafmm_comm_local_create", C.c_int, [C.c_int, C.c_void_p]),
    ("kafmm_comm_destroy", None, [C.c_void_p]),
    ("kafmm_setup_dist_comm", C.c_int, [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                        C.POINTER(C.c_void_p)]),
    ("kafmm_dist_query", C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    ("kafmm_wall_setup", C.c_int, [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    ("kafmm_wall_set_stream", C.c_int, [C.c_void_p, C.c_void_p]),
    ("kafmm_wall_eval", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("kafmm_wall_destroy", None, [C.c_void_p]),
]
EXPORTED = [s[0] for s in _SIGS]


def load_library():
    """Load libkafmm.so (raises if it is missing: there is no fallback)."""
    global _LIB
    if _LIB is None:
        path = lib_path()
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run python -m paper_2010_15155_b200.build)")
        lib = C.CDLL(path)
        for name, res, args in _SIGS:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def _check(st: int, where: str):
    if st != 0:
        lib = load_library()
        raise KafmmError(st, where, (lib.kafmm_last_error() or b"").decode())


def kernel_dims(kernel) -> tuple[int, int]:
    lib = load_library()
    ks, kt = C.c_int(), C.c_int()
    k = KERNELS[kernel] if isinstance(kernel, str) else int(kernel)
    _check(lib.kafmm_kernel_dims(k, C.byref(ks), C.byref(kt)), "kafmm_kernel_dims")
    return ks.value, kt.value


def fp64_peak(which: str = "dmma") -> float:
    """Measured FP64 TFLOP/s of the device: 'dmma' (tensor core) or 'dfma'."""
    lib = load_library()
    v = C.c_double()
    _check(lib.kafmm_fp64_peak(0 if which == "dmma" else 1, C.byref(v)), "kafmm_fp64_peak")
    return v.value


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("kafmm: no CUDA device (there is no CPU fallback)")
    return torch


class KAFMM:
    """A plan: octree, lists and operators for one point set (sources = targets).

    points: (n, 3) float64 in [0,1)^3, numpy array or CUDA tensor.
    """

    def __init__(self, points, kernel: str, p: int, max_pts: int, stream=None):
        torch = _torch()
        self.lib = load_library()
        self.kernel = kernel
        if isinstance(points, np.ndarray):
            pts = torch.from_numpy(np.ascontiguousarray(points, dtype=np.float64)).cuda()
        else:
            pts = points.to(device="cuda", dtype=torch.float64).contiguous()
        self.n = int(pts.shape[0])
        self.k_s, self.k_t = kernel_dims(kernel)
        h = C.c_void_p()
        torch.cuda.synchronize()
        _check(self.lib.kafmm_setup(C.c_void_p(pts.data_ptr()), self.n, KERNELS[kernel], int(p), int(max_pts),
                                    C.byref(h)), "kafmm_setup")
        self.h = h
        if stream is not None:
            self.set_stream(stream)

    def set_stream(self, stream):
        ptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        _check(self.lib.kafmm_set_stream(self.h, C.c_void_p(ptr)), "kafmm_set_stream")

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            self.lib.kafmm_destroy(h)
            self.h = None

    def close(self):
        self.__del__()

    # hot path
    def eval(self, src, out=None):
        """src: (n, k_s) float64 CUDA tensor (user order) -> (n, k_t) CUDA tensor."""
        torch = _torch()
        assert src.is_cuda and src.dtype == torch.float64 and src.shape == (self.n, self.k_s)
        src = src.contiguous()
        if out is None:
            out = torch.empty((self.n, self.k_t), dtype=torch.float64, device=src.device)
        _check(self.lib.kafmm_eval(self.h, C.c_void_p(src.data_ptr()), C.c_void_p(out.data_ptr())), "kafmm_eval")
        return out

    def eval_host(self, src: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """End-to-end through the C ABI with host buffers (copies inside)."""
        assert src.dtype == np.float64 and src.shape == (self.n, self.k_s) and src.flags.c_contiguous
        if out is None:
            out = np.empty((self.n, self.k_t))
        _check(self.lib.kafmm_eval_host(self.h, C.c_void_p(src.ctypes.data), C.c_void_p(out.ctypes.data)),
               "kafmm_eval_host")
        return out

    def check_values(self, src):
        _check(self.lib.kafmm_check_values(self.h, C.c_void_p(src.data_ptr())), "kafmm_check_values")

    def sync(self):
        _check(self.lib.kafmm_sync(self.h), "kafmm_sync")

    # introspection
    def info(self) -> Info:
        inf = Info()
        _check(self.lib.kafmm_get_info(self.h, C.byref(inf)), "kafmm_get_info")
        return inf

    def tree(self) -> dict:
        nb = self.info().n_boxes
        lev = np.empty(nb, np.int32)
        ijk = np.empty((nb, 3), np.int32)
        par = np.empty(nb, np.int32)
        leaf = np.empty(nb, np.int32)
        pb = np.empty(nb, np.int64)
        pe = np.empty(nb, np.int64)
        ptrs = [C.c_void_p(a.ctypes.data) for a in (lev, ijk, par, leaf, pb, pe)]
        _check(self.lib.kafmm_get_tree(self.h, *ptrs), "kafmm_get_tree")
        return dict(level=lev, ijk=ijk, parent=par, leaf=leaf.astype(bool), pbeg=pb, pend=pe)

    def permutation(self) -> np.ndarray:
        perm = np.empty(self.n, np.int64)
        _check(self.lib.kafmm_get_permutation(self.h, C.c_void_p(perm.ctypes.data)), "kafmm_get_permutation")
        return perm

    def lists(self, which: str):
        inf = self.info()
        n = {"U": inf.n_u_pairs, "V": inf.n_v_pairs, "W": inf.n_w_pairs, "X": inf.n_w_pairs}[which]
        tgt = np.empty(max(n, 1), np.int32)
        src = np.empty(max(n, 1), np.int32)
        _check(self.lib.kafmm_get_list(self.h, ord(which), C.c_void_p(tgt.ctypes.data), C.c_void_p(src.ctypes.data)),
               "kafmm_get_list")
        return tgt[:n], src[:n]

    def set_timing(self, on):
        """False/0 off; True/1 per-stage events (serialised); 2 total + M2L product only (overlapped)."""
        _check(self.lib.kafmm_set_timing(self.h, int(on)), "kafmm_set_timing")

    def stage_times(self) -> dict:
        arr = (C.c_float * N_STAGES)()
        _check(self.lib.kafmm_stage_times(self.h, arr), "kafmm_stage_times")
        return {self.lib.kafmm_stage_name(i).decode(): float(arr[i]) for i in range(N_STAGES)}

    M2L_MODES = {"dense": 0, "fft": 1, "fft_blocks": 2, "fft_pairs": 3}

    def set_m2l(self, mode: str):
        """'dense' (FP64 tensor-core GEMMs), 'fft' (lattice convolution, product
        per chunk by block fill), 'fft_blocks' or 'fft_pairs' (forced product)."""
        _check(self.lib.kafmm_set_m2l_mode(self.h, self.M2L_MODES[mode]), "kafmm_set_m2l_mode")

    def m2l(self) -> str:
        m = C.c_int()
        _check(self.lib.kafmm_get_m2l_mode(self.h, C.byref(m)), "kafmm_get_m2l_mode")
        return ["dense", "fft", "fft_blocks", "fft_pairs"][m.value]

    def set_graph(self, on: bool):
        """Replay evaluations from a captured CUDA graph (same src/out pointers)."""
        _check(self.lib.kafmm_set_graph(self.h, int(bool(on))), "kafmm_set_graph")

    def fft_stats(self) -> dict:
        st = np.zeros(10, np.int64)
        _check(self.lib.kafmm_fft_stats(self.h, C.c_void_p(st.ctypes.data)), "kafmm_fft_stats")
        keys = ("chunks", "source_blocks", "target_parents", "targets", "v_pairs", "pair_chunks", "n_freq",
                "budget_bytes", "source_children", "items")
        return {k: int(v) for k, v in zip(keys, st)}

    def launch_count(self) -> int:
        n = C.c_int()
        _check(self.lib.kafmm_launch_count(self.h, C.byref(n)), "kafmm_launch_count")
        return n.value


class KAFMMWall:
    """RPY spheres above a no-slip wall (Table X): particles in
    [0,1)^2 x (1/2, 1), wall at z = 1/2.  eval([f, b]) -> [u, lap u]."""

    def __init__(self, points, p: int, max_pts: int, stream=None):
        torch = _torch()
        self.lib = load_library()
        if isinstance(points, np.ndarray):
            pts = torch.from_numpy(np.ascontiguousarray(points, dtype=np.float64)).cuda()
        else:
            pts = points.to(device="cuda", dtype=torch.float64).contiguous()
        self.n = int(pts.shape[0])
        h = C.c_void_p()
        torch.cuda.synchronize()
        _check(self.lib.kafmm_wall_setup(C.c_void_p(pts.data_ptr()), self.n, int(p), int(max_pts), C.byref(h)),
               "kafmm_wall_setup")
        self.h = h
        if stream is not None:
            ptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
            _check(self.lib.kafmm_wall_set_stream(self.h, C.c_void_p(ptr)), "kafmm_wall_set_stream")

    def eval(self, src, out=None):
        torch = _torch()
        assert src.is_cuda and src.dtype == torch.float64 and src.shape == (self.n, 4)
        src = src.contiguous()
        if out is None:
            out = torch.empty((self.n, 6), dtype=torch.float64, device=src.device)
        _check(self.lib.kafmm_wall_eval(self.h, C.c_void_p(src.data_ptr()), C.c_void_p(out.data_ptr())),
               "kafmm_wall_eval")
        return out

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            self.lib.kafmm_wall_destroy(h)
            self.h = None

    def close(self):
        self.__del__()


class KAFMM2(KAFMM):
    """Separate source and target point sets (kafmm_setup2 / kafmm_eval2):
    eval(src_values (n_src x k_s)) -> (n_trg x k_t) at the target points."""

    def __init__(self, src_points, trg_points, kernel: str, p: int, max_pts: int, stream=None):
        torch = _torch()
        self.lib = load_library()
        self.kernel = kernel
        dev = lambda a: (torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()  # noqa: E731
                         if isinstance(a, np.ndarray) else a.to(device="cuda", dtype=torch.float64).contiguous())
        sp, tp = dev(src_points), dev(trg_points)
        self.n_src, self.n_trg = int(sp.shape[0]), int(tp.shape[0])
        self.n = self.n_src + self.n_trg
        self.k_s, self.k_t = kernel_dims(kernel)
        h = C.c_void_p()
        torch.cuda.synchronize()
        _check(self.lib.kafmm_setup2(C.c_void_p(sp.data_ptr()), self.n_src, C.c_void_p(tp.data_ptr()), self.n_trg,
                                     KERNELS[kernel], int(p), int(max_pts), C.byref(h)), "kafmm_setup2")
        self.h = h
        if stream is not None:
            self.set_stream(stream)

    def eval(self, src, out=None):
        torch = _torch()
        assert src.is_cuda and src.dtype == torch.float64 and src.shape == (self.n_src, self.k_s)
        src = src.contiguous()
        if out is None:
            out = torch.empty((self.n_trg, self.k_t), dtype=torch.float64, device=src.device)
        _check(self.lib.kafmm_eval2(self.h, C.c_void_p(src.data_ptr()), C.c_void_p(out.data_ptr())), "kafmm_eval2")
        return out


def unique_id() -> bytes:
    """A new NCCL unique id (128 bytes) for kafmm_setup_dist; rank 0 makes it."""
    lib = load_library()
    buf = (C.c_ubyte * 128)()
    _check(lib.kafmm_get_unique_id(buf), "kafmm_get_unique_id")
    return bytes(buf)


class LocalComms:
    """kafmm_comm_local_create: `world` in-process communicators (test transport:
    ranks are host threads of this process on one GPU)."""

    def __init__(self, world: int):
        self.lib = load_library()
        arr = (C.c_void_p * world)()
        _check(self.lib.kafmm_comm_local_create(int(world), arr), "kafmm_comm_local_create")
        self.handles = [C.c_void_p(arr[i]) for i in range(world)]

    def close(self):
        for h in self.handles:
            if h.value:
                self.lib.kafmm_comm_destroy(h)
        self.handles = []

    def __del__(self):
        if getattr(self, "handles", None):
            self.close()


DIST_KEYS = ("rank", "world", "n_global", "n_caller", "n_owned", "n_local", "n_ghost_points", "n_rows",
             "n_ghost_boxes", "n_shared", "plan_bytes", "bytes_per_eval", "n_v_local", "n_p2p_local")


class DistKAFMM(KAFMM):
    """One rank of a partitioned plan (kafmm_setup_dist over NCCL, or
    kafmm_setup_dist_comm over a LocalComms handle).  eval takes and returns
    this caller's rows; all ranks must call it collectively."""

    def __init__(self, local_points, kernel: str, p: int, max_pts: int, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, comm=None, stream=None):
        torch = _torch()
        self.lib = load_library()
        self.kernel = kernel
        if isinstance(local_points, np.ndarray):
            pts = torch.from_numpy(np.ascontiguousarray(local_points, dtype=np.float64).reshape(-1, 3)).cuda()
        else:
            pts = local_points.to(device="cuda", dtype=torch.float64).contiguous().reshape(-1, 3)
        self.n = int(pts.shape[0])
        self.k_s, self.k_t = kernel_dims(kernel)
        h = C.c_void_p()
        ptr = C.c_void_p(pts.data_ptr()) if self.n > 0 else C.c_void_p(0)
        torch.cuda.synchronize()
        if comm is not None:
            _check(self.lib.kafmm_setup_dist_comm(ptr, self.n, KERNELS[kernel], int(p), int(max_pts), comm,
                                                  C.byref(h)), "kafmm_setup_dist_comm")
        else:
            idb = (C.c_ubyte * 128).from_buffer_copy(nccl_id)
            _check(self.lib.kafmm_setup_dist(ptr, self.n, KERNELS[kernel], int(p), int(max_pts), int(rank),
                                             int(world), idb, C.byref(h)), "kafmm_setup_dist")
        self.h = h
        if stream is not None:
            self.set_stream(stream)

    def eval(self, src, out=None):
        torch = _torch()
        assert src.is_cuda and src.dtype == torch.float64 and src.shape == (self.n, self.k_s)
        src = src.contiguous()
        if out is None:
            out = torch.empty((self.n, self.k_t), dtype=torch.float64, device=src.device)
        sp = C.c_void_p(src.data_ptr()) if src.numel() else C.c_void_p(8)
        op = C.c_void_p(out.data_ptr()) if out.numel() else C.c_void_p(8)
        _check(self.lib.kafmm_eval(self.h, sp, op), "kafmm_eval")
        return out

    def dist_info(self) -> dict:
        v = np.zeros(len(DIST_KEYS), np.int64)
        _check(self.lib.kafmm_dist_query(self.h, 0, C.c_void_p(v.ctypes.data)), "kafmm_dist_query")
        d = {k: int(x) for k, x in zip(DIST_KEYS, v)}
        w = d["world"]
        cuts = np.zeros(w + 1, np.int64)
        _check(self.lib.kafmm_dist_query(self.h, 1, C.c_void_p(cuts.ctypes.data)), "kafmm_dist_query")
        cnt = np.zeros(6 * w, np.int64)
        _check(self.lib.kafmm_dist_query(self.h, 2, C.c_void_p(cnt.ctypes.data)), "kafmm_dist_query")
        d["cuts"] = cuts
        for i, k in enumerate(("val_send", "val_recv", "ue_send", "ue_recv", "out_send", "out_recv")):
            d[k] = cnt[i * w:(i + 1) * w]
        return d
