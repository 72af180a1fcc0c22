"""paper_2008_00216_b200 -- B200-native fused-gate state-vector engine.

Thin ctypes binding over the C ABI in include/sv.h (argument marshalling
only: planning runs in the native library, every step of the state update
runs in its sm_100a kernels).  PyTorch only provides device memory (the
state tensor), the CUDA stream and torch.distributed bootstrap.

There is NO CPU fallback: if libstv.so is missing or no CUDA device is
present, constructing a State raises.
"""
from __future__ import annotations

import ctypes
import json
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("STV_LIB") or os.path.join(_HERE, "libstv.so")   # STV_LIB: A/B builds (tools)

KINDS = {"h": 0, "x": 1, "y": 2, "z": 3, "s": 4, "t": 5, "sx": 6, "sy": 7, "sw": 8,
         "cz": 9, "cnot": 10, "swap": 11, "cphase": 12, "fsim": 13, "u1": 14, "u2": 15}
GATE_ADJOINT = 0x1
OPT_PROFILE, OPT_NO_RELABEL, OPT_NO_REORDER, OPT_ONE_GATE, OPT_NO_DIAG_FOLD, OPT_NO_GROUPS = 1, 2, 4, 8, 16, 32
OPT_NO_VARIANTS = 128
OPT_NO_TC, OPT_NO_PLAN_CACHE, OPT_NO_SINK, OPT_TMA = 256, 512, 1024, 2048
C64, C128 = 0, 1
STATUS = {0: "SV_OK", 1: "SV_ERR_INVALID_ARG", 2: "SV_ERR_OUT_OF_MEMORY", 3: "SV_ERR_CUDA",
          4: "SV_ERR_NCCL", 5: "SV_ERR_UNSUPPORTED", 6: "SV_ERR_STATE"}
PASS_KINDS = ["tile", "tile_low", "tile_high", "diag", "cnot", "remap", "init", "other"]

# every entry point declared in include/sv.h
EXPORTS = ["sv_create", "sv_wrap", "sv_create_dist", "sv_create_virtual", "sv_set_basis",
           "sv_set_uniform", "sv_apply_circuit", "sv_get_amplitudes", "sv_read_state", "sv_norm", "sv_sample",
           "sv_last_run_stats", "sv_get_frame", "sv_plan_json", "sv_plan_blob", "sv_remap_peers", "sv_destroy",
           "sv_last_error", "sv_version"]


class SvError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Gate(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("q0", ctypes.c_int32), ("q1", ctypes.c_int32),
                ("theta", ctypes.c_double), ("phi", ctypes.c_double),
                ("m", ctypes.POINTER(ctypes.c_double))]


class Options(ctypes.Structure):
    _fields_ = [("kmax", ctypes.c_int32), ("tile_bits", ctypes.c_int32), ("low_bits", ctypes.c_int32),
                ("budget", ctypes.c_int32), ("flags", ctypes.c_uint32)]


class Stats(ctypes.Structure):
    _fields_ = [("plan_ms", ctypes.c_double), ("run_ms", ctypes.c_double),
                ("n_pass", ctypes.c_int32 * 8), ("pass_ms", ctypes.c_double * 8),
                ("alg_bytes", ctypes.c_double), ("remap_bytes", ctypes.c_double),
                ("n_ops", ctypes.c_int32 * 4), ("n_kernels", ctypes.c_int32), ("h2d_bytes", ctypes.c_double),
                ("alg_flops", ctypes.c_double), ("tc_flops", ctypes.c_double),
                ("n_tc_pass", ctypes.c_int32), ("n_tc_steps", ctypes.c_int32)]


_lib = None


def lib():
    """Load libstv.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2008_00216_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        vp, u64, sz = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_size_t
        L.sv_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
        L.sv_wrap.argtypes = [ctypes.c_int, ctypes.c_int, vp, sz, vp, ctypes.POINTER(vp)]
        L.sv_create_dist.argtypes = [ctypes.c_int, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, vp, sz, vp,
                                     ctypes.POINTER(vp)]
        L.sv_create_virtual.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
        L.sv_set_basis.argtypes = [vp, u64]
        L.sv_set_uniform.argtypes = [vp]
        L.sv_apply_circuit.argtypes = [vp, ctypes.POINTER(Gate), sz, ctypes.POINTER(Options)]
        L.sv_get_amplitudes.argtypes = [vp, ctypes.POINTER(u64), u64, sz, vp]
        L.sv_read_state.argtypes = [vp, u64, u64, vp]
        L.sv_norm.argtypes = [vp, ctypes.POINTER(ctypes.c_double)]
        L.sv_sample.argtypes = [vp, u64, sz, ctypes.POINTER(u64)]
        L.sv_last_run_stats.argtypes = [vp, ctypes.POINTER(Stats)]
        L.sv_get_frame.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(u64)]
        L.sv_plan_json.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(Gate), sz,
                                   ctypes.POINTER(Options), ctypes.c_char_p, sz, ctypes.POINTER(sz)]
        L.sv_plan_blob.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(Gate), sz,
                                   ctypes.POINTER(Options), ctypes.c_void_p, sz, ctypes.POINTER(sz),
                                   ctypes.POINTER(ctypes.c_uint32), sz, ctypes.POINTER(sz)]
        L.sv_remap_peers.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint32, ctypes.c_int,
                                     ctypes.POINTER(ctypes.c_int32)]
        L.sv_destroy.argtypes = [vp]
        L.sv_last_error.restype = ctypes.c_char_p
        L.sv_version.restype = ctypes.c_char_p
        for f in EXPORTS:
            if f not in ("sv_last_error", "sv_version"):
                getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(code):
    if code != 0:
        raise SvError(code, lib().sv_last_error().decode())


def _angle(a):
    num, den = a
    return float(num) * math.pi / float(den)


def marshal(gates):
    """(name, qubits, params) tuples -> sv_gate array (+ keep-alive list)."""
    arr = (Gate * max(1, len(gates)))()
    keep = []
    for i, (name, qs, p) in enumerate(gates):
        adj = name.endswith("_dg")
        base = name[:-3] if adj else name
        g = arr[i]
        g.kind = KINDS[base]
        g.flags = GATE_ADJOINT if adj else 0
        g.q0 = qs[0]
        g.q1 = qs[1] if len(qs) > 1 else -1
        g.theta = g.phi = 0.0
        if base == "cphase":
            g.phi = _angle(p[0])
        elif base == "fsim":
            g.theta, g.phi = _angle(p[0]), _angle(p[1])
        if base in ("u1", "u2"):
            m = (ctypes.c_double * len(p))(*p)
            keep.append(m)
            g.m = ctypes.cast(m, ctypes.POINTER(ctypes.c_double))
        else:
            g.m = None
    return arr, keep


def options(kmax=0, tile_bits=0, low_bits=0, budget=0, flags=0, profile=False):
    o = Options()
    o.kmax, o.tile_bits, o.low_bits, o.budget = kmax, tile_bits, low_bits, budget
    o.flags = flags | (OPT_PROFILE if profile else 0)
    return o


def plan_json(n, gates, n_global=0, dtype="c64", **kw):
    """Host-only: the plan the engine would run (no GPU needed)."""
    arr, keep = marshal(gates)
    o = options(**kw)
    need = ctypes.c_size_t(0)
    L = lib()
    dt = C64 if dtype == "c64" else C128
    rc = L.sv_plan_json(n, n_global, dt, arr, len(gates), ctypes.byref(o), None, 0, ctypes.byref(need))
    if rc != 0 and need.value == 0:
        _check(rc)
    buf = ctypes.create_string_buffer(need.value)
    _check(L.sv_plan_json(n, n_global, dt, arr, len(gates), ctypes.byref(o), buf, need.value,
                          ctypes.byref(need)))
    return json.loads(buf.value.decode())


def plan_blob(n, gates, n_global=0, dtype="c64", **kw):
    """Host-only: (blob bytes, pass offsets) of the encoded device plan."""
    arr, keep = marshal(gates)
    o = options(**kw)
    need, npass = ctypes.c_size_t(0), ctypes.c_size_t(0)
    L = lib()
    dt = C64 if dtype == "c64" else C128
    L.sv_plan_blob(n, n_global, dt, arr, len(gates), ctypes.byref(o), None, 0, ctypes.byref(need), None, 0,
                   ctypes.byref(npass))
    buf = ctypes.create_string_buffer(max(1, need.value))
    offs = (ctypes.c_uint32 * max(1, npass.value))()
    _check(L.sv_plan_blob(n, n_global, dt, arr, len(gates), ctypes.byref(o), buf, need.value, ctypes.byref(need),
                          offs, npass.value, ctypes.byref(npass)))
    return bytes(buf.raw[:need.value]), list(offs)[:npass.value]


def remap_peers(g, rank, gbits, m):
    out = (ctypes.c_int32 * (1 << m))()
    _check(lib().sv_remap_peers(g, rank, gbits, m, out))
    return list(out)


class State:
    """A 2^n complex state vector on the current CUDA device.

    dtype 'c64' (interleaved float32 pairs, the paper's choice, PAPER.md
    L355-358) or 'c128'.  The buffer is a torch tensor on the current device;
    kernels run on torch's current stream.  `virtual_g > 0` emulates a
    2^g-rank partition on one GPU (global-qubit remaps as device copies).
    """

    def __init__(self, n: int, dtype: str = "c64", virtual_g: int = 0, dist=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("State needs a CUDA device (no CPU fallback)")
        L = lib()
        self.n, self.dtype = n, dtype
        self.dt = C64 if dtype == "c64" else C128
        self._h = ctypes.c_void_p()
        self.tensor = None
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        if dist is not None:
            rank, world, uid = dist["rank"], dist["world"], dist["uid"]
            g = world.bit_length() - 1
            real = torch.float32 if dtype == "c64" else torch.float64
            self.tensor = torch.empty(2 << (n - g), dtype=real, device="cuda")
            nbytes = self.tensor.numel() * self.tensor.element_size()
            ub = (ctypes.c_char * 128).from_buffer_copy(bytes(uid))
            _check(L.sv_create_dist(n, self.dt, ub, rank, world, ctypes.c_void_p(self.tensor.data_ptr()),
                                    nbytes, stream, ctypes.byref(self._h)))
        elif virtual_g:
            _check(L.sv_create_virtual(n, self.dt, virtual_g, ctypes.byref(self._h)))
        else:
            real = torch.float32 if dtype == "c64" else torch.float64
            self.tensor = torch.empty(2 << n, dtype=real, device="cuda")
            nbytes = self.tensor.numel() * self.tensor.element_size()
            _check(L.sv_wrap(n, self.dt, ctypes.c_void_p(self.tensor.data_ptr()), nbytes, stream,
                             ctypes.byref(self._h)))

    # -- lifecycle -------------------------------------------------------
    def close(self):
        if self._h:
            lib().sv_destroy(self._h)
            self._h = ctypes.c_void_p()
        self.tensor = None        # release the torch-owned buffer with the state

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- the four north-star calls -----------------------------------------
    def set_basis(self, x: int = 0):
        _check(lib().sv_set_basis(self._h, x))

    def set_uniform(self):
        _check(lib().sv_set_uniform(self._h))

    def apply(self, gates, **kw):
        arr, keep = marshal(gates)
        o = options(**kw)
        _check(lib().sv_apply_circuit(self._h, arr, len(gates), ctypes.byref(o)))
        return self

    def apply_marshalled(self, arr, ng, o):
        _check(lib().sv_apply_circuit(self._h, arr, ng, ctypes.byref(o)))

    def amplitudes(self, idx=None, first=0, count=None):
        """complex128 numpy array of amplitudes at logical indices."""
        if idx is not None:
            idx = np.ascontiguousarray(idx, dtype=np.uint64)
            count = idx.size
            out = np.empty(count, dtype=np.complex128)
            _check(lib().sv_get_amplitudes(self._h, idx.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), 0,
                                           count, out.ctypes.data))
            return out
        if count is None:
            count = (1 << self.n) - first
        out = np.empty(count, dtype=np.complex128)
        _check(lib().sv_get_amplitudes(self._h, None, first, count, out.ctypes.data))
        return out

    def read_state(self, first=0, count=None, out=None):
        """Raw readout in the state's dtype (complex64 / complex128) in logical order."""
        if count is None:
            count = (1 << self.n) - first
        if out is None:
            out = np.empty(count, dtype=np.complex64 if self.dtype == "c64" else np.complex128)
        _check(lib().sv_read_state(self._h, first, count, ctypes.c_void_p(out.ctypes.data)
                                   if isinstance(out, np.ndarray) else ctypes.c_void_p(out)))
        return out

    def norm(self) -> float:
        v = ctypes.c_double()
        _check(lib().sv_norm(self._h, ctypes.byref(v)))
        return v.value

    def sample(self, shots: int, seed: int = 0):
        """Logical basis indices drawn from |a|^2 (include/sv.h sv_sample), uint64 numpy array."""
        out = np.zeros(max(1, shots), dtype=np.uint64)
        _check(lib().sv_sample(self._h, seed, shots, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
        return out[:shots]

    def stats(self) -> dict:
        s = Stats()
        _check(lib().sv_last_run_stats(self._h, ctypes.byref(s)))
        return {"plan_ms": s.plan_ms, "run_ms": s.run_ms,
                "n_pass": dict(zip(PASS_KINDS, list(s.n_pass))),
                "pass_ms": dict(zip(PASS_KINDS, list(s.pass_ms))),
                "alg_bytes": s.alg_bytes, "remap_bytes": s.remap_bytes,
                "n_ops": dict(zip(["dense", "diag", "cnot", "group"], list(s.n_ops))),
                "n_kernels": s.n_kernels, "h2d_bytes": s.h2d_bytes, "alg_flops": s.alg_flops,
                "tc_flops": s.tc_flops, "n_tc_pass": s.n_tc_pass, "n_tc_steps": s.n_tc_steps}

    def frame(self):
        perm = (ctypes.c_int32 * 64)()
        xm = ctypes.c_uint64()
        _check(lib().sv_get_frame(self._h, perm, ctypes.byref(xm)))
        return list(perm)[: self.n], xm.value


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId from the NCCL torch loaded (for sv_create_dist)."""
    import torch  # noqa: F401  (loads torch's libnccl.so.2)
    nccl = ctypes.CDLL("libnccl.so.2", mode=ctypes.RTLD_GLOBAL)
    uid = (ctypes.c_char * 128)()
    rc = nccl.ncclGetUniqueId(uid)
    if rc != 0:
        raise SvError(4, f"ncclGetUniqueId failed ({rc})")
    return bytes(uid)


def version():
    return lib().sv_version().decode()
