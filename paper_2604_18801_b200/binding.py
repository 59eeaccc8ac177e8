"""ctypes binding of libcc (include/cc.h).  Same names as the C ABI; torch tensors in, torch
tensors out.  Marshalling only."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import asdict, dataclass

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
# CC_LIB_PATH: load another build of libcc (development A/B measurements only)
_LIB_PATH = os.environ.get("CC_LIB_PATH") or os.path.join(HERE, "libcc.so")

CC_OK, CC_NOT_CONVERGED = 0, 2
CC_ORIG, CC_DECOMP, CC_CORR = 0, 1, 2
STOP_ACTIVE, STOP_EPS, STOP_NONE, STOP_RESTORED = 0, 1, 2, 3
CC_RUN_HOST = 1
_STATUS = {0: "CC_OK", 2: "CC_NOT_CONVERGED", 64: "CC_E_ARG", 65: "CC_E_DATA", 66: "CC_E_BOUND",
           67: "CC_E_OOM", 68: "CC_E_CUDA", 69: "CC_E_NCCL", 70: "CC_E_STATE"}


class CCError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class _Params(C.Structure):
    _fields_ = [("box", C.c_double), ("periodic", C.c_int), ("b", C.c_double), ("eta", C.c_double),
                ("xi", C.c_double), ("m", C.c_int), ("alpha", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps_adam", C.c_double), ("t_max", C.c_int), ("eps_loss", C.c_double),
                ("stop_mode", C.c_int), ("optimizer", C.c_int), ("vanilla_step", C.c_double),
                ("graph_batch", C.c_int), ("cells_per_particle", C.c_double), ("profile", C.c_int),
                ("frontier", C.c_int), ("alloc_fn", C.c_void_p), ("free_fn", C.c_void_p), ("alloc_user", C.c_void_p)]


_ALLOC_T = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
_FREE_T = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class _Dist(C.Structure):
    _fields_ = [("rank", C.c_int), ("nranks", C.c_int), ("nccl_id_h", C.c_void_p), ("vgroup", C.c_void_p)]


class _VP(C.Structure):
    _fields_ = [("n_pairs", C.c_int64), ("n_editable", C.c_int64), ("n_linked", C.c_int64),
                ("n_violated0", C.c_int64), ("n_local", C.c_int64), ("cells_per_axis", C.c_int64),
                ("b", C.c_double)]


class _Corr(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("active0", C.c_int64), ("active_final", C.c_int64),
                ("loss0", C.c_double), ("loss_final", C.c_double), ("converged", C.c_int), ("pad", C.c_int),
                ("violated0", C.c_int64), ("violated_final", C.c_int64)]


class _Mcc(C.Structure):
    _fields_ = [("tp", C.c_uint64), ("tn", C.c_uint64), ("fp", C.c_uint64), ("fn", C.c_uint64), ("mcc", C.c_double)]


class _Th(C.Structure):
    _fields_ = [(k, C.c_float) for k in ("xi_f", "xip_f", "b2", "lo2", "hi2", "c_b", "c_f", "Lf", "hLf", "lo2s_i",
                                         "hi2s_i", "lo2s_w", "hi2s_w")] + \
               [("pad", C.c_int)] + [(k, C.c_double) for k in ("b", "eps_q", "mu", "r_search", "r_link")] + \
               [("near_pairs", C.c_int64)]


class _Run(C.Structure):
    _fields_ = [("vp", _VP), ("corr", _Corr)]


EXPORTS = ["cc_default_params", "cc_nccl_unique_id", "cc_create", "cc_destroy", "cc_last_error", "cc_build_cells",
           "cc_find_vulnerable", "cc_get_pairs", "cc_correct", "cc_get_trace", "cc_get_schedule", "cc_fof_label", "cc_mcc",
           "cc_halo_sizes", "cc_hmf", "cc_kernel_stats", "cc_run", "cc_edit_encode", "cc_edit_decode",
           "cc_get_thresholds", "cc_vgroup_create", "cc_vgroup_destroy", "cc_edit_pack", "cc_edit_unpack"]

_lib = None


def lib_path() -> str:
    return _LIB_PATH


def lib():
    """Load libcc.so (building it with nvcc if it is missing).  Raises if it cannot."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        from .build import build
        build()
    L = C.CDLL(_LIB_PATH)
    P = C.POINTER
    vp, f, u32, i64, d = C.c_void_p, C.c_float, C.c_uint32, C.c_int64, C.c_double
    L.cc_default_params.argtypes = [P(_Params)]
    L.cc_default_params.restype = None
    L.cc_nccl_unique_id.argtypes = [vp]
    L.cc_create.argtypes = [P(vp), C.c_int, vp, P(_Params), P(_Dist)]
    L.cc_destroy.argtypes = [vp]
    L.cc_destroy.restype = None
    L.cc_last_error.argtypes = [vp]
    L.cc_last_error.restype = C.c_char_p
    L.cc_build_cells.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp, vp]
    L.cc_find_vulnerable.argtypes = [vp, P(_VP)]
    L.cc_get_pairs.argtypes = [vp, vp, vp, vp, i64, P(i64)]
    L.cc_correct.argtypes = [vp, vp, vp, vp, P(_Corr)]
    L.cc_get_trace.argtypes = [vp, P(i64), P(d), P(i64), i64, P(i64)]
    L.cc_get_schedule.argtypes = [vp, P(i64), i64, P(i64)]
    L.cc_fof_label.argtypes = [vp, C.c_int, vp, P(i64)]
    L.cc_mcc.argtypes = [vp, C.c_int, P(_Mcc)]
    L.cc_halo_sizes.argtypes = [vp, C.c_int, i64, P(i64), i64, P(i64)]
    L.cc_hmf.argtypes = [P(i64), i64, d, C.c_int, d, d, P(d), P(d)]
    L.cc_kernel_stats.argtypes = [vp, C.c_char_p, i64, P(d), P(i64), i64, P(i64), C.c_int]
    L.cc_run.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_int, P(_Run)]
    L.cc_edit_encode.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, P(i64)]
    L.cc_edit_decode.argtypes = [vp, i64, vp, vp, vp, vp, vp, i64, vp, vp, vp]
    L.cc_get_thresholds.argtypes = [vp, P(_Th)]
    L.cc_vgroup_create.argtypes = [C.c_int, P(vp)]
    L.cc_edit_pack.argtypes = [vp, vp, i64, vp, i64, P(i64)]
    L.cc_edit_unpack.argtypes = [vp, vp, i64, vp]
    L.cc_vgroup_destroy.argtypes = [vp]
    L.cc_vgroup_destroy.restype = None
    for name in EXPORTS:
        if name not in ("cc_default_params", "cc_destroy", "cc_last_error", "cc_vgroup_destroy"):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L


@dataclass
class Params:
    """cc_params (include/cc.h): Alg. 1 REQUIRE line plus box and perf knobs."""
    box: float = 1.0
    periodic: int = 1
    b: float = 0.0
    eta: float = 0.2
    xi: float = 0.0
    m: int = 16
    alpha: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps_adam: float = 1e-8
    t_max: int = 10000
    eps_loss: float = 1e-10
    stop_mode: int = STOP_ACTIVE
    optimizer: int = 0
    vanilla_step: float = 0.0
    graph_batch: int = 16
    cells_per_particle: float = 0.03
    profile: int = 0
    frontier: int = 1
    torch_allocator: bool = False  # scratch from torch's caching allocator (cc_params.alloc_fn)

    def to_c(self) -> _Params:
        return _Params(**{k: v for k, v in asdict(self).items() if k != "torch_allocator"})


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _check_dev(t, dtype, name):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name}: expected a CUDA tensor (no CPU path exists)")
    if t.dtype != dtype or not t.is_contiguous():
        raise TypeError(f"{name}: expected contiguous {dtype}")


class Corrector:
    """One context of libcc on one GPU (cc_create).  Methods map 1:1 to the C ABI."""

    def __init__(self, params: Params, device: int | None = None, stream: torch.cuda.Stream | None = None,
                 dist: tuple | None = None):
        if not torch.cuda.is_available():
            raise CCError(68, "no CUDA device: libcc has no CPU path")
        self.lib = lib()
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.params = params
        self._p = params.to_c()
        if params.torch_allocator:  # scratch from torch's caching allocator, on this context's stream
            dev, st = self.device, self.stream

            def _alloc(nbytes, user):
                try:
                    return torch.cuda.caching_allocator_alloc(int(nbytes), dev, st)
                except Exception:
                    return None

            def _free(ptr, user):
                torch.cuda.caching_allocator_delete(ptr)

            self._cb = (_ALLOC_T(_alloc), _FREE_T(_free))  # kept alive with the context
            self._p.alloc_fn = C.cast(self._cb[0], C.c_void_p)
            self._p.free_fn = C.cast(self._cb[1], C.c_void_p)
        self._d = None
        if dist is not None:
            # (rank, nranks, nccl unique id) for NCCL ranks, or (rank, nranks, None, VGroup)
            rank, nranks, uid = dist[:3]
            vg = dist[3] if len(dist) > 3 else None
            self._uid = C.create_string_buffer(bytes(uid), 128) if uid is not None else None
            self._d = _Dist(rank, nranks, C.cast(self._uid, C.c_void_p) if uid is not None else None,
                            vg.h if vg is not None else None)
        h = C.c_void_p()
        st = self.lib.cc_create(C.byref(h), self.device, C.c_void_p(self.stream.cuda_stream), C.byref(self._p),
                                None if self._d is None else C.byref(self._d))
        if st != 0:
            raise CCError(st, "cc_create failed")
        self.h = h
        self.n = 0

    def close(self):
        if getattr(self, "h", None):
            self.lib.cc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, st, ok=(0,)):
        if st not in ok:
            raise CCError(st, self.lib.cc_last_error(self.h).decode(errors="replace"))
        return st

    # S1
    def build_cells(self, x, y, z, xh, yh, zh, gid=None):
        for nm, t in zip("x y z xh yh zh".split(), (x, y, z, xh, yh, zh)):
            _check_dev(t, torch.float32, nm)
        if gid is not None:
            _check_dev(gid, torch.int32, "gid (int32 view of uint32 ids)")
        n = x.shape[0]
        self._inputs = (x, y, z, xh, yh, zh, gid)  # keep alive until the stream is done
        self._chk(self.lib.cc_build_cells(self.h, n, *[_ptr(t) for t in (x, y, z, xh, yh, zh)], _ptr(gid)))
        self.n = n

    def thresholds(self) -> dict:
        """S0 values in use (cc_get_thresholds)."""
        t = _Th()
        self._chk(self.lib.cc_get_thresholds(self.h, C.byref(t)))
        return {k: getattr(t, k) for k, _ in _Th._fields_ if k != "pad"}

    # S2 + S3
    def find_vulnerable(self) -> dict:
        info = _VP()
        self._chk(self.lib.cc_find_vulnerable(self.h, C.byref(info)))
        return {k: getattr(info, k) for k, _ in _VP._fields_}

    def get_pairs(self):
        n = C.c_int64()
        self._chk(self.lib.cc_get_pairs(self.h, None, None, None, 0, C.byref(n)))
        k = n.value
        dev = torch.device("cuda", self.device)
        gi = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
        gj = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
        fl = torch.empty(max(k, 1), dtype=torch.uint8, device=dev)
        self._chk(self.lib.cc_get_pairs(self.h, _ptr(gi), _ptr(gj), _ptr(fl), k, C.byref(n)))
        return gi[:k], gj[:k], fl[:k]

    # S4 + S5
    def correct(self, out=None):
        dev = torch.device("cuda", self.device)
        if out is None:
            out = tuple(torch.empty(self.n, dtype=torch.float32, device=dev) for _ in range(3))
        info = _Corr()
        st = self._chk(self.lib.cc_correct(self.h, *[_ptr(t) for t in out], C.byref(info)), ok=(0, 2))
        d = {k: getattr(info, k) for k, _ in _Corr._fields_ if k != "pad"}
        d["converged"] = bool(d["converged"])
        d["status"] = st
        return out, d

    def trace(self):
        n = C.c_int64()
        a = np.zeros(self.params.t_max + 2, np.int64)
        l = np.zeros(self.params.t_max + 2, np.float64)
        v = np.zeros(self.params.t_max + 2, np.int64)
        self._chk(self.lib.cc_get_trace(self.h, a.ctypes.data_as(C.POINTER(C.c_int64)),
                                        l.ctypes.data_as(C.POINTER(C.c_double)),
                                        v.ctypes.data_as(C.POINTER(C.c_int64)), a.shape[0], C.byref(n)))
        return a[: n.value], l[: n.value], v[: n.value]

    def schedule(self):
        """K3 schedule per iteration: (editables processed, left awake, moved row entries, full
        replay steps, proven-still replay steps, device time in ns at the iteration's end)."""
        n = C.c_int64()
        a = np.zeros((self.params.t_max + 1, 6), np.int64)
        self._chk(self.lib.cc_get_schedule(self.h, a.ctypes.data_as(C.POINTER(C.c_int64)), a.shape[0], C.byref(n)))
        return a[: n.value]

    # f1 edit log (Alg. 1 l.11-13)
    def edit_encode(self, x, y, z, xh0, yh0, zh0, xc, yc, zc, cap=None):
        """(flags u8[ceil(3n/8)], q int64[n_edits]) of Delta = corrected - decompressed;
        x, y, z = the original positions (bound-safe indices, R32)."""
        for nm, t in zip("x y z xh0 yh0 zh0 xc yc zc".split(), (x, y, z, xh0, yh0, zh0, xc, yc, zc)):
            _check_dev(t, torch.float32, nm)
        n = xh0.shape[0]
        dev = torch.device("cuda", self.device)
        nbytes = (3 * n + 7) // 8
        flags = torch.empty(max((nbytes + 3) // 4, 1), dtype=torch.int32, device=dev).view(torch.uint8)[:nbytes]
        ne = C.c_int64()
        args = [_ptr(t) for t in (x, y, z, xh0, yh0, zh0, xc, yc, zc)]
        if cap is None:  # count first (CC_E_OOM with cap 0 reports n_edits), then an exact-size q
            self._chk(self.lib.cc_edit_encode(self.h, n, *args, _ptr(flags), None, 0, C.byref(ne)), ok=(0, 67))
            cap = ne.value
        q = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
        self._chk(self.lib.cc_edit_encode(self.h, n, *args, _ptr(flags), _ptr(q), cap, C.byref(ne)))
        return flags, (q if ne.value == q.shape[0] else q[: ne.value].clone())

    def edit_decode(self, xh0, yh0, zh0, flags, q, out=None):
        """x_rec = x_hat0 + scatter(dequantise(q), flags)."""
        for nm, t in zip("xh0 yh0 zh0".split(), (xh0, yh0, zh0)):
            _check_dev(t, torch.float32, nm)
        _check_dev(flags, torch.uint8, "flags")
        _check_dev(q, torch.int64, "q")
        n = xh0.shape[0]
        dev = torch.device("cuda", self.device)
        for nm, t in (("yh0", yh0), ("zh0", zh0)):
            if t.shape[0] != n:
                raise ValueError(f"{nm}: length {t.shape[0]} != {n}")
        if flags.numel() < (3 * n + 7) // 8:
            raise ValueError(f"flags: {flags.numel()} bytes < ceil(3n/8) = {(3 * n + 7) // 8}")
        for nm, t in (("xh0", xh0), ("flags", flags), ("q", q)):
            if t.device != dev:
                raise ValueError(f"{nm}: on {t.device}, the context is on {dev}")
        if out is None:
            out = tuple(torch.empty(n, dtype=torch.float32, device=dev) for _ in range(3))
        for k, t in enumerate(out):
            _check_dev(t, torch.float32, f"out[{k}]")
            if t.numel() < n or t.device != dev:
                raise ValueError(f"out[{k}]: needs {n} floats on {dev}")
        self._chk(self.lib.cc_edit_decode(self.h, n, *[_ptr(t) for t in (xh0, yh0, zh0)], _ptr(flags), _ptr(q),
                                          q.shape[0], *[_ptr(t) for t in out]))
        return out

    def edit_pack(self, q):
        """(m+2)-bit packing of the edit indices (Alg. 1 l.13, R33) -> int32 view of the u32 words."""
        _check_dev(q, torch.int64, "q")
        n = q.shape[0]
        nw = C.c_int64()
        self._chk(self.lib.cc_edit_pack(self.h, _ptr(q), n, None, 0, C.byref(nw)), ok=(0, 67))
        words = torch.empty(max(nw.value, 1), dtype=torch.int32, device=q.device)
        self._chk(self.lib.cc_edit_pack(self.h, _ptr(q), n, _ptr(words), nw.value, C.byref(nw)))
        return words[: nw.value]

    def edit_unpack(self, words, n_edits: int):
        _check_dev(words, torch.int32, "words (int32 view of u32)")
        q = torch.empty(max(n_edits, 1), dtype=torch.int64, device=words.device)
        self._chk(self.lib.cc_edit_unpack(self.h, _ptr(words), n_edits, _ptr(q)))
        return q[:n_edits]

    # S6
    def fof_label(self, which=CC_ORIG, labels=None):
        if labels is None:
            labels = torch.empty(max(self.n, 1), dtype=torch.int32, device=torch.device("cuda", self.device))[: self.n]
        ng = C.c_int64()
        self._chk(self.lib.cc_fof_label(self.h, which, _ptr(labels), C.byref(ng)))
        return labels, ng.value

    # S7
    def mcc(self, which=CC_CORR) -> dict:
        m = _Mcc()
        self._chk(self.lib.cc_mcc(self.h, which, C.byref(m)))
        return {k: getattr(m, k) for k, _ in _Mcc._fields_}

    def halo_sizes(self, which=CC_ORIG, min_size=20) -> np.ndarray:
        n = C.c_int64()
        self._chk(self.lib.cc_halo_sizes(self.h, which, min_size, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), np.int64)
        self._chk(self.lib.cc_halo_sizes(self.h, which, min_size, out.ctypes.data_as(C.POINTER(C.c_int64)),
                                         out.shape[0], C.byref(n)))
        return out[: n.value]

    def kernel_stats(self, reset=True) -> dict:
        names = C.create_string_buffer(8192)
        ms = np.zeros(64, np.float64)
        ln = np.zeros(64, np.int64)
        n = C.c_int64()
        self._chk(self.lib.cc_kernel_stats(self.h, names, 8192, ms.ctypes.data_as(C.POINTER(C.c_double)),
                                           ln.ctypes.data_as(C.POINTER(C.c_int64)), 64, C.byref(n), int(reset)))
        keys = names.value.decode().split("\n")[: n.value]
        return {k: (float(ms[i]), int(ln[i])) for i, k in enumerate(keys)}

    # end-to-end through the ABI (host or device buffers)
    def run(self, x, y, z, xh, yh, zh, out, gid=None, host=False) -> dict:
        info = _Run()
        ptrs = [_ptr(t) for t in (x, y, z, xh, yh, zh)]
        st = self._chk(self.lib.cc_run(self.h, x.shape[0], *ptrs, _ptr(gid), *[_ptr(t) for t in out],
                                       CC_RUN_HOST if host else 0, C.byref(info)), ok=(0, 2))
        self.n = x.shape[0]
        vp = {k: getattr(info.vp, k) for k, _ in _VP._fields_}
        co = {k: getattr(info.corr, k) for k, _ in _Corr._fields_ if k != "pad"}
        return {"vp": vp, "corr": co, "status": st}


class VGroup:
    """cc_vgroup_create: an in-process group of virtual ranks sharing one GPU (cc_dist.vgroup).
    Each rank's Corrector must be driven by its own thread; close every Corrector first."""

    def __init__(self, nranks: int):
        h = C.c_void_p()
        st = lib().cc_vgroup_create(nranks, C.byref(h))
        if st != 0:
            raise CCError(st, "cc_vgroup_create")
        self.h = h
        self.nranks = nranks

    def close(self):
        if getattr(self, "h", None):
            lib().cc_vgroup_destroy(self.h)
            self.h = None


def nccl_unique_id() -> bytes:
    """cc_nccl_unique_id: 128 bytes for cc_dist.nccl_id_h (rank 0 creates, all ranks share)."""
    buf = C.create_string_buffer(128)
    st = lib().cc_nccl_unique_id(buf)
    if st != 0:
        raise CCError(st, "cc_nccl_unique_id")
    return buf.raw


def slab_of(x: torch.Tensor, nranks: int, box: float) -> torch.Tensor:
    """Owner rank of each original x under the x-slab decomposition of cc_dist (rank r owns
    [r L/R, (r+1) L/R)) -- the same fp64 rule the library checks."""
    r = torch.floor(x.double() * (nranks / box)).long()
    r = torch.clamp(r, 0, nranks - 1)
    # guard the fp64 boundary rounding: re-test against the exact slab edges
    lo = box * r.double() / nranks
    hi = box * (r + 1).double() / nranks
    xd = x.double()
    r = torch.where(xd < lo, r - 1, torch.where(xd >= hi, r + 1, r))
    return torch.clamp(r, 0, nranks - 1)


def shell_masks(x: torch.Tensor, rank: int, nranks: int, box: float, gw: float):
    """Owned particles sent as ghosts (§III-D): (to the left rank, to the right rank) =
    (x < lo + gw, x >= hi - gw) for the slab [lo, hi) of `rank` -- the rule of dist.cu's
    k_shell_flags, exposed for the host-side protocol tests."""
    lo = box * rank / nranks
    hi = box * (rank + 1) / nranks
    xd = x.double()
    return xd < lo + gw, xd >= hi - gw


def hmf(sizes, vol: float, n_bins: int = 50, lo: float = 0.0, hi: float = 0.0):
    """cc_hmf: dn/dlog10 M of a halo catalogue; lo >= hi: the catalogue's range."""
    s = np.ascontiguousarray(np.asarray(sizes, dtype=np.int64))
    e = np.zeros(n_bins + 1, np.float64)
    d = np.zeros(n_bins, np.float64)
    st = lib().cc_hmf(s.ctypes.data_as(C.POINTER(C.c_int64)), s.shape[0], vol, n_bins, lo, hi,
                      e.ctypes.data_as(C.POINTER(C.c_double)), d.ctypes.data_as(C.POINTER(C.c_double)))
    if st != 0:
        raise CCError(st, "cc_hmf")
    return e, d
