"""paper_1103_4697_b200 -- B200-native multi-modular elimination for curvetop.

Python mirror of the reference's elimination API (namespace ``curvetop``,
/root/reference/proj/include/curvetop/elim.hpp) over the C ABI of
``libctg.so`` (include/ctg.h).  Same names, argument meaning and error
behaviour as the reference:

=============================  ==========================================  =========================
this module                    reference                                   C ABI
=============================  ==========================================  =========================
``resultant(p, q, var)``       ``curvetop::resultant`` elim.cpp:95-136     ``ctg_resultant``
``yun_squarefree(p)``          ``curvetop::yun_squarefree`` elim.cpp:138   ``ctg_yun_squarefree``
``gcd_univariate(p, q)``       ``curvetop::gcd_univariate`` elim.cpp:80    ``ctg_gcd_univariate``
``square_free_part(p)``        ``curvetop::square_free_part`` elim.cpp:204 ``ctg_square_free_part``
=============================  ==========================================  =========================

Polynomials: bivariate = ``{(deg_x, deg_y): int}``, univariate = list of ints
(low -> high).  ``PreconditionError`` / ``Error`` mirror the reference's
exception types (numeric.hpp:15-30).  Every computation runs on the GPU;
without a CUDA device (or without the built library) the calls raise -- there
is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CTG_LIBRARY") or os.path.join(_PKG, "libctg.so")  # CTG_LIBRARY: A/B experiments


class Error(RuntimeError):
    """curvetop::Error (numeric.hpp:15-18)."""


class PreconditionError(Error):
    """curvetop::PreconditionError (numeric.hpp:20-24)."""


class CudaError(Error):
    """A CUDA failure or no device: libctg has no CPU fallback."""


class UnsupportedError(Error):
    """CTG_UNSUPPORTED: outside the library's GPU path (message says which limit)."""


CTG_OK, CTG_PRECONDITION, CTG_INVALID, CTG_UNSUPPORTED, CTG_INTERNAL, CTG_CUDA = range(6)

_i32p = C.POINTER(C.c_int32)
_i8p = C.POINTER(C.c_int8)
_u32p = C.POINTER(C.c_uint32)


class _Bipoly(C.Structure):
    _fields_ = [("n_terms", C.c_int32), ("dx", _i32p), ("dy", _i32p), ("sign", _i8p), ("limb_off", _u32p),
                ("limbs", _u32p)]


class _Upoly(C.Structure):
    _fields_ = [("n_coeffs", C.c_int32), ("sign", _i8p), ("limb_off", _u32p), ("limbs", _u32p)]


class _UpolyBuf(C.Structure):
    _fields_ = [("n_coeffs", C.c_int32), ("sign", _i8p), ("limb_off", _u32p), ("limbs", _u32p)]


class _BipolyBuf(C.Structure):
    _fields_ = [("n_terms", C.c_int32), ("dx", _i32p), ("dy", _i32p), ("sign", _i8p), ("limb_off", _u32p),
                ("limbs", _u32p)]


class _SqfBuf(C.Structure):
    _fields_ = [("unit_sign", C.c_int8), ("unit_nlimbs", C.c_int32), ("unit_limbs", _u32p), ("n_factors", C.c_int32),
                ("mult", _i32p), ("factors", C.POINTER(_UpolyBuf))]


class _Opts(C.Structure):
    _fields_ = [("device", C.c_int32), ("verify", C.c_int32), ("n_devices", C.c_int32), ("reserved0", C.c_int32),
                ("devices", _i32p), ("comm", C.c_void_p)]


class CallStats(C.Structure):
    _fields_ = [("total_ms", C.c_double), ("setup_ms", C.c_double), ("h2d_ms", C.c_double), ("device_ms", C.c_double),
                ("d2h_ms", C.c_double), ("decode_ms", C.c_double), ("h2d_bytes", C.c_int64),
                ("d2h_bytes", C.c_int64), ("n_primes", C.c_int32), ("n_points", C.c_int32),
                ("n_coeffs", C.c_int32), ("out_limbs", C.c_int32), ("kernel_launches", C.c_int32),
                ("flagged_units", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class PlanInfo(C.Structure):
    _fields_ = [("n_primes", C.c_int32), ("n_points", C.c_int32), ("n_coeffs", C.c_int32), ("out_limbs", C.c_int32),
                ("deg_p", C.c_int32), ("deg_q", C.c_int32), ("derivative", C.c_int32), ("trivial", C.c_int32),
                ("bound_bits", C.c_double), ("work_mulmods", C.c_double), ("h2d_bytes", C.c_int64),
                ("batch", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# Every symbol include/ctg.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "ctg_resultant", "ctg_yun_squarefree", "ctg_gcd_univariate", "ctg_square_free_part", "ctg_upoly_free",
    "ctg_sqf_free", "ctg_last_error", "ctg_abi_version", "ctg_device_count", "ctg_last_call_stats",
    "ctg_plan_create", "ctg_plan_get_info", "ctg_plan_upload", "ctg_plan_residues", "ctg_plan_crt",
    "ctg_plan_decode", "ctg_plan_check", "ctg_plan_launches", "ctg_plan_destroy", "ctg_plan_stage",
    "ctg_microbench_int", "ctg_plan_crt_sharded", "ctg_resultant_batch", "ctg_plan_create_batch",
    "ctg_plan_stage_batch", "ctg_plan_crt_batch", "ctg_upoly_free_batch", "ctg_gcd_bivariate", "ctg_bipoly_free",
    "ctg_comm_unique_id", "ctg_comm_init_rank", "ctg_comm_destroy", "ctg_comm_all_gather",
    "ctg_yun_squarefree_batch", "ctg_modp_gcd_degree", "ctg_comm_all_to_all", "ctg_plan_interp_cols",
    "ctg_plan_crt_cols",
)

_lib = None
_lock = threading.Lock()


def lib():
    """Load libctg.so (built by ``paper_1103_4697_b200.build``); raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_1103_4697_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.ctg_resultant.argtypes = [C.POINTER(_Bipoly), C.POINTER(_Bipoly), C.c_int32, C.POINTER(_UpolyBuf),
                                    C.POINTER(_Opts)]
        L.ctg_yun_squarefree.argtypes = [C.POINTER(_Upoly), C.POINTER(_SqfBuf), C.POINTER(_Opts)]
        L.ctg_gcd_univariate.argtypes = [C.POINTER(_Upoly), C.POINTER(_Upoly), C.POINTER(_UpolyBuf),
                                         C.POINTER(_Opts)]
        L.ctg_square_free_part.argtypes = [C.POINTER(_Upoly), C.POINTER(_UpolyBuf), C.POINTER(_Opts)]
        L.ctg_upoly_free.argtypes = [C.POINTER(_UpolyBuf)]
        L.ctg_upoly_free_batch.argtypes = [C.POINTER(_UpolyBuf), C.c_int32]
        L.ctg_sqf_free.argtypes = [C.POINTER(_SqfBuf)]
        L.ctg_gcd_bivariate.argtypes = [C.POINTER(_Bipoly), C.POINTER(_Bipoly), C.POINTER(_BipolyBuf),
                                        C.POINTER(_Opts)]
        L.ctg_bipoly_free.argtypes = [C.POINTER(_BipolyBuf)]
        L.ctg_last_error.restype = C.c_char_p
        L.ctg_last_call_stats.argtypes = [C.POINTER(CallStats)]
        L.ctg_plan_create.argtypes = [C.POINTER(_Bipoly), C.POINTER(_Bipoly), C.c_int32, C.POINTER(_Opts),
                                      C.POINTER(C.c_void_p)]
        L.ctg_plan_get_info.argtypes = [C.c_void_p, C.POINTER(PlanInfo)]
        L.ctg_plan_upload.argtypes = [C.c_void_p, C.c_void_p]
        L.ctg_plan_residues.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]
        L.ctg_plan_stage.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]
        L.ctg_microbench_int.argtypes = [C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]
        L.ctg_modp_gcd_degree.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                          C.POINTER(C.c_int32), C.POINTER(C.c_uint32), C.POINTER(C.c_float),
                                          C.POINTER(_Opts)]
        L.ctg_plan_crt.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]
        L.ctg_plan_crt_sharded.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                           C.c_void_p, C.c_void_p]
        L.ctg_resultant_batch.argtypes = [C.c_int32, C.POINTER(_Bipoly), C.POINTER(_Bipoly), C.c_int32,
                                          C.POINTER(_UpolyBuf), C.POINTER(_Opts)]
        L.ctg_plan_create_batch.argtypes = [C.c_int32, C.POINTER(_Bipoly), C.POINTER(_Bipoly), C.c_int32,
                                            C.POINTER(_Opts), C.POINTER(C.c_void_p)]
        L.ctg_plan_stage_batch.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int64,
                                           C.c_void_p]
        L.ctg_plan_crt_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int64, C.c_int32,
                                         C.c_int32, C.c_void_p, C.c_void_p]
        L.ctg_plan_decode.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_UpolyBuf)]
        L.ctg_plan_check.argtypes = [C.c_void_p, C.c_void_p]
        L.ctg_plan_launches.argtypes = [C.c_void_p]
        L.ctg_plan_destroy.argtypes = [C.c_void_p]
        L.ctg_yun_squarefree_batch.argtypes = [C.c_int32, C.POINTER(_Upoly), C.POINTER(_SqfBuf), C.POINTER(_Opts)]
        L.ctg_comm_unique_id.argtypes = [C.c_void_p]
        L.ctg_comm_init_rank.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)]
        L.ctg_comm_destroy.argtypes = [C.c_void_p]
        L.ctg_comm_all_gather.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
        L.ctg_comm_all_to_all.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
        L.ctg_plan_interp_cols.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_int32,
                                           C.c_int32, C.c_void_p, C.c_void_p]
        L.ctg_plan_crt_cols.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                        C.c_void_p]
        _lib = L
        return L


def _raise(status: int, what: str):
    msg = lib().ctg_last_error().decode(errors="replace") or what
    if status == CTG_PRECONDITION:
        raise PreconditionError(msg)
    if status == CTG_CUDA:
        raise CudaError(msg)
    if status == CTG_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise Error(msg)


def _check(status: int, what: str):
    if status != CTG_OK:
        _raise(status, what)


# ----------------------------------------------------------------------------
# Marshaling: Python ints <-> sign + little-endian u32 limbs (CSR)
# ----------------------------------------------------------------------------

def _encode_ints(values):
    n = len(values)
    sign = np.zeros(n, dtype=np.int8)
    off = np.zeros(n + 1, dtype=np.uint32)
    chunks = []
    pos = 0
    for i, v in enumerate(values):
        if v:
            mag = -v if v < 0 else v
            sign[i] = -1 if v < 0 else 1
            nl = (mag.bit_length() + 31) >> 5
            chunks.append(mag.to_bytes(nl * 4, "little"))
            pos += nl
        off[i + 1] = pos
    limbs = np.frombuffer(b"".join(chunks), dtype=np.uint32) if chunks else np.zeros(1, dtype=np.uint32)
    return sign, off, np.ascontiguousarray(limbs)


class HostBipoly:
    """Caller-owned host buffers of one bivariate operand (kept alive with the struct)."""

    def __init__(self, f: dict):
        items = sorted((k, v) for k, v in f.items() if v)
        self.dx = np.array([k[0] for k, _ in items], dtype=np.int32)
        self.dy = np.array([k[1] for k, _ in items], dtype=np.int32)
        self.sign, self.off, self.limbs = _encode_ints([v for _, v in items])
        self.struct = _Bipoly(len(items), self.dx.ctypes.data_as(_i32p), self.dy.ctypes.data_as(_i32p),
                              self.sign.ctypes.data_as(_i8p), self.off.ctypes.data_as(_u32p),
                              self.limbs.ctypes.data_as(_u32p))
        self.nbytes = self.dx.nbytes + self.dy.nbytes + self.sign.nbytes + self.off.nbytes + self.limbs.nbytes

    @classmethod
    def from_terms(cls, terms, pad_limbs: int = 0):
        """Raw CSR operand from [(dx, dy, value), ...] in the given order -- duplicates,
        explicit zeros and ``pad_limbs`` high zero limbs per term are kept (the library
        must sum / drop / trim them like the reference's map insertion)."""
        self = cls.__new__(cls)
        n = len(terms)
        self.dx = np.array([t[0] for t in terms], dtype=np.int32)
        self.dy = np.array([t[1] for t in terms], dtype=np.int32)
        self.sign = np.zeros(n, dtype=np.int8)
        self.off = np.zeros(n + 1, dtype=np.uint32)
        chunks, pos = [], 0
        for i, (_, _, v) in enumerate(terms):
            mag = -v if v < 0 else v
            self.sign[i] = -1 if v < 0 else (1 if v > 0 else 0)
            nl = (mag.bit_length() + 31) >> 5
            nl += pad_limbs if v else 0
            chunks.append(mag.to_bytes(nl * 4, "little"))
            pos += nl
            self.off[i + 1] = pos
        raw = b"".join(chunks)
        self.limbs = np.ascontiguousarray(np.frombuffer(raw, dtype=np.uint32) if raw else np.zeros(1, np.uint32))
        self.struct = _Bipoly(n, self.dx.ctypes.data_as(_i32p), self.dy.ctypes.data_as(_i32p),
                              self.sign.ctypes.data_as(_i8p), self.off.ctypes.data_as(_u32p),
                              self.limbs.ctypes.data_as(_u32p))
        self.nbytes = self.dx.nbytes + self.dy.nbytes + self.sign.nbytes + self.off.nbytes + self.limbs.nbytes
        return self


class HostUpoly:
    def __init__(self, p):
        self.sign, self.off, self.limbs = _encode_ints(list(p))
        self.struct = _Upoly(len(p), self.sign.ctypes.data_as(_i8p), self.off.ctypes.data_as(_u32p),
                             self.limbs.ctypes.data_as(_u32p))


def _decode_buf(buf: _UpolyBuf) -> list:
    n = buf.n_coeffs
    if n == 0:
        return []
    off = np.ctypeslib.as_array(buf.limb_off, shape=(n + 1,))
    total = int(off[n])
    sign = np.ctypeslib.as_array(buf.sign, shape=(n,))
    raw = bytes(np.ctypeslib.as_array(buf.limbs, shape=(max(total, 1),)).tobytes()) if total else b""
    out = []
    for i in range(n):
        a, b = int(off[i]) * 4, int(off[i + 1]) * 4
        v = int.from_bytes(raw[a:b], "little")
        out.append(-v if sign[i] < 0 else v)
    return out


def _opts(device, devices=None, comm=None):
    """ctg_opts: one device (default), a prime-sharded device list (one process; repeats allowed),
    or a multi-process Comm."""
    o = _Opts()
    o.device = -1 if device is None else int(device)
    o.verify = 1
    if devices is not None and len(devices) > 1:
        o._devs = (C.c_int32 * len(devices))(*[int(d) for d in devices])  # kept alive with the struct
        o.n_devices = len(devices)
        o.devices = C.cast(o._devs, _i32p)
    if comm is not None:
        o.comm = comm.handle
    return o


class Comm:
    """A multi-process communicator (ctg_comm): rank `rank` of `nranks`, on `device`.
    ``Comm.unique_id()`` on rank 0, share the bytes (e.g. torch.distributed.broadcast_object_list),
    then ``Comm(nranks, rank, uid, device)`` on every rank."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib().ctg_comm_unique_id(buf), "comm_unique_id")
        return bytes(buf)

    def __init__(self, nranks: int, rank: int, uid: bytes, device: int):
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().ctg_comm_init_rank(nranks, rank, buf, device, C.byref(h)), "comm_init_rank")
        self.handle, self.nranks, self.rank, self.device = h, nranks, rank, device

    def all_gather(self, send_ptr, recv_ptr, words, stream=0):
        _check(lib().ctg_comm_all_gather(self.handle, C.c_void_p(send_ptr), C.c_void_p(recv_ptr), words,
                                         C.c_void_p(stream)), "comm_all_gather")

    def all_to_all(self, send_ptr, recv_ptr, words, stream=0):
        """Block r of send (words u32) to rank r; block s of recv from rank s."""
        _check(lib().ctg_comm_all_to_all(self.handle, C.c_void_p(send_ptr), C.c_void_p(recv_ptr), words,
                                         C.c_void_p(stream)), "comm_all_to_all")

    def close(self):
        if self.handle:
            lib().ctg_comm_destroy(self.handle)
            self.handle = None


def last_call_stats() -> dict:
    s = CallStats()
    lib().ctg_last_call_stats(C.byref(s))
    return s.as_dict()


def microbench_int(device=None) -> dict:
    """Measured integer-pipe peaks (results/s): IMAD, IMAD.WIDE, Montgomery two-product reductions."""
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    _check(lib().ctg_microbench_int(-1 if device is None else int(device), C.byref(a), C.byref(b), C.byref(c)),
           "microbench")
    return {"imad_per_s": a.value, "imad_wide_per_s": b.value, "mmul2_per_s": c.value}


def uni_prime(prime_index: int = 0, device=None, method: int = 0) -> int:
    """The prime_index-th univariate (K6) prime, or with method=2 the prime_index-th (0..2)
    square-freeness probe prime (< 2^15)."""
    z = (C.c_uint32 * 1)(0)
    p, d = C.c_uint32(), C.c_int32()
    _check(lib().ctg_modp_gcd_degree(z, 0, z, 0, int(prime_index), int(method), C.byref(d), C.byref(p), None,
                                     _opts(device)), "modp_gcd_degree")
    return p.value


def modp_gcd_degree(a, b, prime_index: int = 0, method: int = 0, device=None) -> dict:
    """deg gcd(a mod p, b mod p) over F_p for p = uni_prime(prime_index) (K6 test / A-B hook,
    ``ctg_modp_gcd_degree``); a, b: integer coefficients, ascending.  method 0 = the blocked
    Lehmer kernel, 1 = one pass per Euclid step, 2 = the blocked kernel in the probe's 32-bit
    arithmetic modulo the prime_index-th probe prime (< 2^15).  Returns {"deg", "prime", "ms"}."""
    p = uni_prime(prime_index, device, method if method == 2 else 0)
    A = (C.c_uint32 * len(a))(*[int(v) % p for v in a])
    B = (C.c_uint32 * len(b))(*[int(v) % p for v in b])
    d, pp, ms = C.c_int32(), C.c_uint32(), C.c_float()
    _check(lib().ctg_modp_gcd_degree(A, len(a) - 1, B, len(b) - 1, int(prime_index), int(method), C.byref(d),
                                     C.byref(pp), C.byref(ms), _opts(device)), "modp_gcd_degree")
    return {"deg": d.value, "prime": pp.value, "ms": ms.value}


def device_count() -> int:
    return int(lib().ctg_device_count())


# ----------------------------------------------------------------------------
# The reference-facing API
# ----------------------------------------------------------------------------

def resultant_host(p: HostBipoly, q: HostBipoly, var: str = "y", device=None) -> list:
    """ctg_resultant on pre-marshaled host operands (the e2e benchmark path)."""
    out = _UpolyBuf()
    o = _opts(device)
    _check(lib().ctg_resultant(C.byref(p.struct), C.byref(q.struct), 1 if var in ("x", "X") else 0, C.byref(out),
                               C.byref(o)), "resultant")
    try:
        return _decode_buf(out)
    finally:
        lib().ctg_upoly_free(C.byref(out))


def resultant_raw(p: HostBipoly, q: HostBipoly, var: str = "y", device=None) -> int:
    """ctg_resultant into a library buffer that is freed again (no Python-int decoding):
    the C-ABI call a C/C++ caller makes.  Returns the number of result coefficients."""
    out = _UpolyBuf()
    o = _opts(device)
    _check(lib().ctg_resultant(C.byref(p.struct), C.byref(q.struct), 1 if var in ("x", "X") else 0, C.byref(out),
                               C.byref(o)), "resultant")
    n = out.n_coeffs
    lib().ctg_upoly_free(C.byref(out))
    return n


def yun_squarefree_raw(p: HostUpoly, device=None) -> list:
    """ctg_yun_squarefree into library buffers that are freed again (no Python-int decoding):
    the C-ABI call a C/C++ caller (the drop-in TU) makes.  Returns [(degree, multiplicity)]."""
    out = _SqfBuf()
    o = _opts(device)
    _check(lib().ctg_yun_squarefree(C.byref(p.struct), C.byref(out), C.byref(o)), "yun_squarefree")
    try:
        return [(int(out.factors[i].n_coeffs) - 1, int(out.mult[i])) for i in range(out.n_factors)]
    finally:
        lib().ctg_sqf_free(C.byref(out))


class HostBatch:
    """Caller-owned host operands of a batch of resultants (arrays of ctg_bipoly)."""

    def __init__(self, pairs):
        self.ops = [(HostBipoly(p), HostBipoly(q)) for p, q in pairs]
        n = len(self.ops)
        self.p = (_Bipoly * max(1, n))(*[a.struct for a, _ in self.ops])
        self.q = (_Bipoly * max(1, n))(*[b.struct for _, b in self.ops])
        self.n = n
        self.nbytes = sum(a.nbytes + b.nbytes for a, b in self.ops)


def resultant_batch_raw(hb: HostBatch, var: str = "y", device=None, devices=None, comm=None) -> int:
    """ctg_resultant_batch into library buffers that are freed again (the C/C++ caller's call)."""
    outs = (_UpolyBuf * max(1, hb.n))()
    o = _opts(device, devices, comm)
    _check(lib().ctg_resultant_batch(hb.n, hb.p, hb.q, 1 if var in ("x", "X") else 0, outs, C.byref(o)),
           "resultant_batch")
    total = sum(outs[i].n_coeffs for i in range(hb.n))
    lib().ctg_upoly_free_batch(outs, hb.n)
    return total


def resultant_batch(pairs, var: str = "y", device=None, devices=None, comm=None) -> list:
    """[res(p, q) for (p, q) in pairs] with one batched GPU pipeline per input shape; with
    `devices` (list of ordinals, repeats allowed) or `comm` (multi-process) the primes are
    sharded over several GPUs (ctg_opts.n_devices / ctg_opts.comm)."""
    hb = HostBatch(pairs)
    outs = (_UpolyBuf * max(1, hb.n))()
    o = _opts(device, devices, comm)
    _check(lib().ctg_resultant_batch(hb.n, hb.p, hb.q, 1 if var in ("x", "X") else 0, outs, C.byref(o)),
           "resultant_batch")
    res = []
    for i in range(hb.n):
        try:
            res.append(_decode_buf(outs[i]))
        finally:
            lib().ctg_upoly_free(C.byref(outs[i]))
    return res


def resultant(p: dict, q: dict, var: str = "y", device=None) -> list:
    """res(p, q) eliminating ``var`` -- curvetop::resultant (elim.hpp:30-31).

    Conventions (elim.hpp:24-29): both zero -> PreconditionError; one zero -> [];
    both of degree 0 in var -> [1]; degree-0 operand q -> q^deg(p).
    """
    return resultant_host(HostBipoly(p), HostBipoly(q), var, device)


def gcd_bivariate(f: dict, g: dict, device=None) -> dict:
    """curvetop::gcd_bivariate (elim.hpp:42, elim.cpp:178-202): a modular coprimality probe,
    and Brown's modular bivariate gcd (certified) when the primitive parts share a factor."""
    hf, hg = HostBipoly(f), HostBipoly(g)
    out = _BipolyBuf()
    o = _opts(device)
    _check(lib().ctg_gcd_bivariate(C.byref(hf.struct), C.byref(hg.struct), C.byref(out), C.byref(o)),
           "gcd_bivariate")
    try:
        n = out.n_terms
        res = {}
        if n:
            off = np.ctypeslib.as_array(out.limb_off, shape=(n + 1,))
            total = int(off[n])
            raw = bytes(np.ctypeslib.as_array(out.limbs, shape=(max(total, 1),)).tobytes()) if total else b""
            for t in range(n):
                v = int.from_bytes(raw[int(off[t]) * 4:int(off[t + 1]) * 4], "little")
                res[(int(out.dx[t]), int(out.dy[t]))] = -v if out.sign[t] < 0 else v
        return res
    finally:
        lib().ctg_bipoly_free(C.byref(out))


def yun_squarefree(p: list, device=None):
    """curvetop::yun_squarefree (elim.hpp:34): returns (unit, [(factor, multiplicity), ...])."""
    hp = HostUpoly(p)
    out = _SqfBuf()
    o = _opts(device)
    _check(lib().ctg_yun_squarefree(C.byref(hp.struct), C.byref(out), C.byref(o)), "yun_squarefree")
    try:
        unit = 0
        if out.unit_nlimbs:
            limbs = np.ctypeslib.as_array(out.unit_limbs, shape=(out.unit_nlimbs,))
            unit = int.from_bytes(limbs.tobytes(), "little")
        unit = -unit if out.unit_sign < 0 else unit
        factors = []
        for i in range(out.n_factors):
            factors.append((_decode_buf(out.factors[i]), int(out.mult[i])))
        return unit, factors
    finally:
        lib().ctg_sqf_free(C.byref(out))


def _decode_sqf(out):
    unit = 0
    if out.unit_nlimbs:
        limbs = np.ctypeslib.as_array(out.unit_limbs, shape=(out.unit_nlimbs,))
        unit = int.from_bytes(limbs.tobytes(), "little")
    unit = -unit if out.unit_sign < 0 else unit
    return unit, [(_decode_buf(out.factors[i]), int(out.mult[i])) for i in range(out.n_factors)]


class HostUpolyBatch:
    """Caller-owned host operands of a batch of univariate inputs (array of ctg_upoly)."""

    def __init__(self, polys):
        self.hs = [HostUpoly(p) for p in polys]
        self.n = len(self.hs)
        self.arr = (_Upoly * max(1, self.n))(*[h.struct for h in self.hs])


def yun_squarefree_batch(polys, device=None, raw=False):
    """[yun_squarefree(p) for p in polys] through ctg_yun_squarefree_batch (one probe launch for
    all inputs).  `polys` may be a HostUpolyBatch (pre-marshaled).  raw=True: (degree,
    multiplicity) patterns only, without decoding the factors."""
    hb = polys if isinstance(polys, HostUpolyBatch) else HostUpolyBatch(polys)
    n, arr = hb.n, hb.arr
    outs = (_SqfBuf * max(1, n))()
    o = _opts(device)
    _check(lib().ctg_yun_squarefree_batch(n, arr, outs, C.byref(o)), "yun_squarefree_batch")
    try:
        if raw:
            return [[(int(outs[b].factors[i].n_coeffs) - 1, int(outs[b].mult[i])) for i in range(outs[b].n_factors)]
                    for b in range(n)]
        return [_decode_sqf(outs[b]) for b in range(n)]
    finally:
        for b in range(n):
            lib().ctg_sqf_free(C.byref(outs[b]))


def gcd_univariate(p: list, q: list, device=None) -> list:
    """curvetop::gcd_univariate (upoly.hpp:92): primitive gcd with positive leading coefficient."""
    hp, hq = HostUpoly(p), HostUpoly(q)
    out = _UpolyBuf()
    o = _opts(device)
    _check(lib().ctg_gcd_univariate(C.byref(hp.struct), C.byref(hq.struct), C.byref(out), C.byref(o)),
           "gcd_univariate")
    try:
        return _decode_buf(out)
    finally:
        lib().ctg_upoly_free(C.byref(out))


def square_free_part(p: list, device=None) -> list:
    """curvetop::square_free_part (elim.hpp:45)."""
    hp = HostUpoly(p)
    out = _UpolyBuf()
    o = _opts(device)
    _check(lib().ctg_square_free_part(C.byref(hp.struct), C.byref(out), C.byref(o)), "square_free_part")
    try:
        return _decode_buf(out)
    finally:
        lib().ctg_upoly_free(C.byref(out))


# ----------------------------------------------------------------------------
# Staged plans (device-resident timing, prime sharding across GPUs)
# ----------------------------------------------------------------------------

class Plan:
    """A ``ctg_plan``: fixed primes / points / CRT constants for one resultant.

    Device buffers are provided by the caller as raw pointers (e.g. torch tensors'
    ``data_ptr()``); streams as raw ``cudaStream_t`` handles (``stream.cuda_stream``).
    """

    def __init__(self, p: dict, q: dict = None, var: str = "y", device=None):
        """Plan(p, q) for one resultant, or Plan(pairs) for a batch of same-shape resultants."""
        self._h = C.c_void_p()
        o = _opts(device)
        elim = 1 if var in ("x", "X") else 0
        if q is None:
            self._hb = HostBatch(p)
            _check(lib().ctg_plan_create_batch(self._hb.n, self._hb.p, self._hb.q, elim, C.byref(o),
                                               C.byref(self._h)), "plan_create_batch")
        else:
            self._hb = HostBatch([(p, q)])
            _check(lib().ctg_plan_create(self._hb.p, self._hb.q, elim, C.byref(o), C.byref(self._h)), "plan_create")
        info = PlanInfo()
        _check(lib().ctg_plan_get_info(self._h, C.byref(info)), "plan_info")
        self.info = info.as_dict()

    def upload(self, stream=0):
        _check(lib().ctg_plan_upload(self._h, C.c_void_p(stream)), "plan_upload")

    def residues(self, k0, k1, rows_ptr, stream=0):
        _check(lib().ctg_plan_residues(self._h, k0, k1, C.c_void_p(rows_ptr), C.c_void_p(stream)), "plan_residues")

    def stage(self, stage, k0, k1, rows_ptr, stream=0, curve_stride=0):
        _check(lib().ctg_plan_stage_batch(self._h, stage, k0, k1, C.c_void_p(rows_ptr), curve_stride,
                                          C.c_void_p(stream)), "plan_stage")

    def crt_batch(self, all_ptr, j0, j1, out_ptr, stream=0, curve_stride=0, row_block=0, block_stride=0):
        _check(lib().ctg_plan_crt_batch(self._h, C.c_void_p(all_ptr), curve_stride, row_block, block_stride, j0, j1,
                                        C.c_void_p(out_ptr), C.c_void_p(stream)), "plan_crt_batch")

    def interp_cols(self, k0, k1, rows_ptr, nranks, row_block, send_ptr, stream=0, curve_stride=0):
        """Stage 3 of primes [k0, k1) written by destination rank: send = [nranks][B][row_block][Jb]."""
        _check(lib().ctg_plan_interp_cols(self._h, k0, k1, C.c_void_p(rows_ptr), curve_stride, nranks, row_block,
                                          C.c_void_p(send_ptr), C.c_void_p(stream)), "plan_interp_cols")

    def crt_cols(self, recv_ptr, nranks, rank, row_block, out_ptr, stream=0):
        """K5 of this rank's coefficient columns from recv = [nranks][B][row_block][Jb]."""
        _check(lib().ctg_plan_crt_cols(self._h, C.c_void_p(recv_ptr), nranks, rank, row_block, C.c_void_p(out_ptr),
                                       C.c_void_p(stream)), "plan_crt_cols")

    def crt(self, all_ptr, j0, j1, out_ptr, stream=0):
        _check(lib().ctg_plan_crt(self._h, C.c_void_p(all_ptr), j0, j1, C.c_void_p(out_ptr), C.c_void_p(stream)),
               "plan_crt")

    def crt_sharded(self, all_ptr, row_block, block_stride, j0, j1, out_ptr, stream=0):
        _check(lib().ctg_plan_crt_sharded(self._h, C.c_void_p(all_ptr), row_block, block_stride, j0, j1,
                                          C.c_void_p(out_ptr), C.c_void_p(stream)), "plan_crt_sharded")

    @property
    def h2d_bytes(self) -> int:
        return int(self.info["h2d_bytes"])

    def check(self, stream=0):
        _check(lib().ctg_plan_check(self._h, C.c_void_p(stream)), "plan_check")

    def decode(self, host_words: np.ndarray) -> list:
        host_words = np.ascontiguousarray(host_words, dtype=np.uint32)
        out = _UpolyBuf()
        _check(lib().ctg_plan_decode(self._h, C.c_void_p(host_words.ctypes.data), C.byref(out)), "plan_decode")
        try:
            return _decode_buf(out)
        finally:
            lib().ctg_upoly_free(C.byref(out))

    def decode_batch_raw(self, host_words: np.ndarray) -> int:
        """Decode every curve of a [B][D][W] CRT output into library-owned sign + limb CSR
        buffers (what ctg_resultant_batch hands a C caller) and free them; no Python ints.
        Returns the total limb count (a use of the result)."""
        host_words = np.ascontiguousarray(host_words, dtype=np.uint32)
        nb = host_words.shape[0]
        per = host_words[0].size * 4
        bufs = (_UpolyBuf * nb)()
        base = host_words.ctypes.data
        dec = lib().ctg_plan_decode
        total = 0
        try:
            for bi in range(nb):
                _check(dec(self._h, C.c_void_p(base + bi * per), C.byref(bufs[bi])), "plan_decode")
                n = bufs[bi].n_coeffs
                total += int(bufs[bi].limb_off[n]) if n else 0
        finally:
            lib().ctg_upoly_free_batch(bufs, nb)
        return total

    @property
    def launches(self) -> int:
        return int(lib().ctg_plan_launches(self._h))

    def close(self):
        if self._h:
            lib().ctg_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
