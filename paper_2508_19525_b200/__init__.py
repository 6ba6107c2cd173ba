"""paper_2508_19525_b200 -- B200-native CKKS fused-linear hot path of BLB (arXiv 2508.19525).

Thin Python binding over ``libblb.so`` (the C ABI declared in include/blb.h).
Argument marshalling only: every step of the path runs in the library's sm_100a
kernels; torch supplies device memory and the current CUDA stream.  There is no
CPU fallback -- importing this package without the built library raises.

Residue tensors are ``torch.int64`` holding the raw uint64 bit patterns
(canonical residues < 2^61, so the values are also non-negative int64).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from ._build import SO, build  # noqa: F401
from . import packing  # noqa: F401

__all__ = ["BLBError", "Params", "Ciphertext", "Keys", "MatmulPlan", "lib", "SO"]


class BLBError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("blb status %d: %s" % (status, msg))
        self.status = status


STATUS = {0: "OK", 1: "INVALID_ARG", 2: "PARAM", 3: "MISSING_KEY", 4: "LEVEL", 5: "SCALE", 6: "LAYOUT",
          7: "OVERFLOW", 8: "CUDA", 9: "NOMEM"}
PACK_SPATIAL, PACK_DIAGONAL = 0, 1
OP_ROTATE, OP_RESCALE, OP_MASK, OP_ENCODE = 0, 1, 2, 3


class _Ct(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("level", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("scale", ctypes.c_double)]


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise ImportError("libblb.so is not built (run __graft_entry__.build()); no CPU fallback exists")
        L = ctypes.CDLL(SO)
        vp, i32, u64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double
        ip = ctypes.POINTER(ctypes.c_int)
        sigs = {
            "blb_last_error": ([], ctypes.c_char_p),
            "blb_counters_get": ([vp], None),
            "blb_counters_reset": ([], None),
            "blb_timing_enable": ([ctypes.c_int], None),
            "blb_measure_pipe_peaks": ([ctypes.c_int, vp, vp, vp], ctypes.c_int),
            "blb_timing_reset": ([], None),
            "blb_timing_read": ([ctypes.c_int, vp, vp, vp], ctypes.c_int),
            "blb_prime_chain": ([ctypes.c_int, vp, ctypes.c_int, vp], ctypes.c_int),
            "blb_params_create": ([vp, ctypes.c_int, vp, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int],
                                  ctypes.c_int),
            "blb_params_destroy": ([vp], None),
            "blb_params_query": ([vp, ip, ip, ip, ip, vp, vp], ctypes.c_int),
            "blb_galois_element": ([vp, i32], ctypes.c_uint32),
            "blb_ntt": ([vp, vp, vp, ctypes.c_int, ctypes.c_int, vp], ctypes.c_int),
            "blb_intt": ([vp, vp, vp, ctypes.c_int, ctypes.c_int, vp], ctypes.c_int),
            "blb_encode": ([vp, vp, ctypes.c_int, dbl, ctypes.c_int, vp, vp], ctypes.c_int),
            "blb_decode": ([vp, vp, ctypes.c_int, dbl, vp, vp], ctypes.c_int),
            "blb_keys_create": ([vp, vp], ctypes.c_int),
            "blb_keys_destroy": ([vp], None),
            "blb_keys_add": ([vp, ctypes.c_uint32, vp, vp], ctypes.c_int),
            "blb_keys_has": ([vp, ctypes.c_uint32], ctypes.c_int),
            "blb_keygen": ([vp, ctypes.c_char_p, vp, ctypes.c_int, ctypes.c_int, vp, vp, vp], ctypes.c_int),
            "blb_encrypt": ([vp, vp, vp, ctypes.c_int, ctypes.c_char_p, u64, dbl, vp, vp], ctypes.c_int),
            "blb_decrypt": ([vp, vp, vp, vp, vp], ctypes.c_int),
            "blb_workspace_bytes": ([vp, ctypes.c_int, ctypes.c_int], ctypes.c_size_t),
            "blb_rotate": ([vp, vp, vp, i32, vp, vp, ctypes.c_size_t, vp], ctypes.c_int),
            "blb_rescale": ([vp, vp, vp, vp, ctypes.c_size_t, vp], ctypes.c_int),
            "blb_mul_pt": ([vp, vp, vp, dbl, vp, vp], ctypes.c_int),
            "blb_add": ([vp, vp, vp, vp, vp], ctypes.c_int),
            "blb_sub": ([vp, vp, vp, vp, vp], ctypes.c_int),
            "blb_add_pt": ([vp, vp, vp, vp, vp], ctypes.c_int),
            "blb_drop_level": ([vp, vp, ctypes.c_int, vp, vp], ctypes.c_int),
            "blb_ckks_to_mpc": ([vp, vp, ctypes.c_int, ctypes.c_char_p, u64, vp, vp, vp, ctypes.c_size_t, vp],
                                ctypes.c_int),
            "blb_ckks_to_mpc_rr_workspace_bytes": ([vp, ctypes.c_int], ctypes.c_size_t),
            "blb_ckks_to_mpc_rr": ([vp, vp, vp, ctypes.c_int, ctypes.c_char_p, ctypes.c_char_p, u64, ctypes.c_int, vp, vp,
                                    vp, ctypes.c_size_t, vp], ctypes.c_int),
            "blb_mhp_column_map": ([ctypes.c_int] * 4 + [vp, ip], ctypes.c_int),
            "blb_share_to_rns": ([vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp], ctypes.c_int),
            "blb_mpc_to_ckks": ([vp, vp, vp, ctypes.c_int, vp, ctypes.c_size_t, vp], ctypes.c_int),
            "blb_share_decode": ([vp, vp, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_size_t, vp], ctypes.c_int),
            "blb_share_to_rns128": ([vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp], ctypes.c_int),
            "blb_mpc_to_ckks128": ([vp, vp, vp, ctypes.c_int, vp, ctypes.c_size_t, vp], ctypes.c_int),
            "blb_share_encode": ([vp, vp, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_size_t, vp], ctypes.c_int),
            "blb_matmul_plan_create": ([vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_int, vp], ctypes.c_int),
            "blb_matmul_plan_destroy": ([vp], None),
            "blb_matmul_plan_create_window": ([vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                               vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                               vp], ctypes.c_int),
            "blb_ct_pt_matmul_acc": ([vp, vp, vp, ctypes.c_int, vp, vp, vp, ctypes.c_size_t, vp], ctypes.c_int),
            "blb_ct_pt_matmul_finish": ([vp, vp, vp, ctypes.c_int, ctypes.c_int, dbl, vp, vp, ctypes.c_size_t, vp],
                                        ctypes.c_int),
            "blb_matmul_plan_info": ([vp, ip, ip, ip, ip, ip, ip, ip], ctypes.c_int),
            "blb_matmul_plan_rotations": ([vp, vp, ip], ctypes.c_int),
            "blb_matmul_pt_count": ([vp, ctypes.c_int, ctypes.c_int, ip], ctypes.c_int),
            "blb_matmul_encode_weights": ([vp, vp, ctypes.c_int, ctypes.c_int, vp, vp], ctypes.c_int),
            "blb_matmul_coeff_bytes": ([vp, ctypes.c_int, ctypes.c_int, vp], ctypes.c_int),
            "blb_matmul_encode_coeffs": ([vp, vp, ctypes.c_int, ctypes.c_int, vp, vp], ctypes.c_int),
            "blb_matmul_coeffs_to_pts": ([vp, vp, ctypes.c_int, ctypes.c_int, vp, vp], ctypes.c_int),
            "blb_matmul_pt_bytes": ([vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
            "blb_matmul_workspace_bytes": ([vp, ctypes.c_int], ctypes.c_size_t),
            "blb_ct_pt_matmul": ([vp, vp, vp, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_size_t,
                                  vp], ctypes.c_int),
            "blb_ct_pt_matmul_batch": ([vp, vp, vp, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, vp, vp,
                                        ctypes.c_size_t, vp], ctypes.c_int),
            "blb_f2_workspace_bytes": ([vp, ctypes.c_int], ctypes.c_size_t),
            "blb_mul_relin": ([vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp], ctypes.c_int),
            "blb_mul_relin_batch_workspace_bytes": ([vp, ctypes.c_int, ctypes.c_int], ctypes.c_size_t),
            "blb_mul_pt_rescale_batch_workspace_bytes": ([vp, ctypes.c_int, ctypes.c_int], ctypes.c_size_t),
            "blb_mul_pt_rescale_batch": ([vp, vp, vp, vp, ctypes.c_int, vp, vp, ctypes.c_size_t, vp], ctypes.c_int),
            "blb_mul_relin_batch": ([vp, vp, vp, vp, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_size_t, vp],
                                    ctypes.c_int),
            "blb_rotate_sum": ([vp, vp, vp, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_size_t, vp], ctypes.c_int),
            "blb_broadcast": ([vp, vp, vp, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_size_t, vp], ctypes.c_int),
            "blb_qk_plan_create": ([vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp],
                                   ctypes.c_int),
            "blb_qk_plan_destroy": ([vp], None),
            "blb_qk_plan_info": ([vp, ip, ip, ip, ip, ip, ip, ip], ctypes.c_int),
            "blb_qk_plan_rotations": ([vp, vp, ip], ctypes.c_int),
            "blb_qk_mask_bytes": ([vp], ctypes.c_size_t),
            "blb_qk_encode_masks": ([vp, vp, vp], ctypes.c_int),
            "blb_qk_workspace_bytes": ([vp], ctypes.c_size_t),
            "blb_ct_ct_qk": ([vp, vp, vp, vp, ctypes.c_int, vp, vp, vp, ctypes.c_size_t, vp], ctypes.c_int),
            "blb_qk_plan_create_window": ([vp] + [ctypes.c_int] * 7 + [vp], ctypes.c_int),
            "blb_qk_acc_bytes": ([vp], ctypes.c_size_t),
            "blb_qk_acc_range": ([vp, ctypes.c_int, ctypes.c_int, ip, ip], ctypes.c_int),
            "blb_ct_ct_qk_acc": ([vp, vp, vp, vp, ctypes.c_int, vp, vp, vp, ctypes.c_size_t, vp], ctypes.c_int),
            "blb_ct_ct_qk_finish": ([vp, vp, vp, ctypes.c_int, ctypes.c_int, dbl, dbl, vp, vp, ctypes.c_size_t, vp],
                                    ctypes.c_int),
        }
        for name, (args, res) in sigs.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise BLBError(status, "%s: %s" % (STATUS.get(status, "?"), lib().blb_last_error().decode()))


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor):
    assert t.is_cuda and t.is_contiguous(), "expected a contiguous CUDA tensor"
    return ctypes.c_void_p(t.data_ptr())


def counters() -> dict:
    out = (ctypes.c_uint64 * 8)()
    lib().blb_counters_get(out)
    names = ["launches", "keyswitches", "limb_ntts", "ct_pt_products", "rescales", "masks", "limb_ntts_int"]
    return {n: int(v) for n, v in zip(names, out)}


def reset_counters():
    lib().blb_counters_reset()


TIMING_MAC, TIMING_NTT, TIMING_KS_INNER, TIMING_MASK_MAC, TIMING_TENSOR = 0, 1, 2, 3, 4


def pipe_peaks(device: int = 0) -> dict:
    """Measured IMAD (fma-heavy pipe) and DFMA (FP64 pipe) ops/s of the device (bench denominators)."""
    a, b = ctypes.c_double(), ctypes.c_double()
    _check(lib().blb_measure_pipe_peaks(int(device), ctypes.byref(a), ctypes.byref(b), _stream()))
    return {"imad_per_s": a.value, "dfma_per_s": b.value}


def timing_enable(on: bool = True):
    lib().blb_timing_enable(int(on))


def timing_reset():
    lib().blb_timing_reset()


def timing_read(category: int) -> dict:
    ms, n, by = ctypes.c_double(), ctypes.c_uint64(), ctypes.c_double()
    _check(lib().blb_timing_read(category, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(by)))
    return {"ms": ms.value, "launches": n.value, "alg_bytes": by.value}


def prime_chain(log_n: int, bits) -> list[int]:
    out = (ctypes.c_uint64 * len(bits))()
    _check(lib().blb_prime_chain(log_n, (ctypes.c_int * len(bits))(*bits), len(bits), out))
    return [int(x) for x in out]


def to_numpy_u64(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().contiguous().numpy().view(np.uint64)


def from_numpy_u64(a: np.ndarray, device="cuda") -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).to(device)


class Params:
    """blb_params_create: ring degree N = 2^log_n, chain q, special primes p, dnum."""

    def __init__(self, log_n: int, q, p, dnum: int, device: int | None = None):
        self.device = torch.cuda.current_device() if device is None else device
        qa = (ctypes.c_uint64 * len(q))(*q)
        pa = (ctypes.c_uint64 * len(p))(*p)
        h = ctypes.c_void_p()
        _check(lib().blb_params_create(ctypes.byref(h), log_n, qa, len(q), pa, len(p), dnum, self.device))
        self._h = h
        ln, nq, npp, al = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        mods = (ctypes.c_uint64 * (len(q) + len(p)))()
        psi = (ctypes.c_uint64 * (len(q) + len(p)))()
        _check(lib().blb_params_query(h, ctypes.byref(ln), ctypes.byref(nq), ctypes.byref(npp), ctypes.byref(al),
                                      mods, psi))
        self.log_n, self.K, self.np_, self.alpha = ln.value, nq.value, npp.value, al.value
        self.N, self.n = 1 << self.log_n, 1 << (self.log_n - 1)
        self.moduli = [int(x) for x in mods]
        self.q, self.p = self.moduli[:self.K], self.moduli[self.K:]
        self.psi = [int(x) for x in psi]

    @classmethod
    def from_preset(cls, preset, device=None) -> "Params":
        primes = prime_chain(preset.log_n, list(preset.q_bits) + list(preset.p_bits))
        k = len(preset.q_bits)
        return cls(preset.log_n, primes[:k], primes[k:], preset.dnum, device)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.blb_params_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def galois(self, step: int) -> int:
        return int(lib().blb_galois_element(self._h, step))

    def beta_top(self) -> int:
        return -(-self.K // self.alpha)

    def empty(self, *shape) -> torch.Tensor:
        return torch.empty(*shape, dtype=torch.int64, device="cuda")

    def workspace(self, op: int, level: int) -> torch.Tensor:
        nbytes = lib().blb_workspace_bytes(self._h, op, level)
        return torch.empty(max(nbytes, 8) // 8 + 1, dtype=torch.int64, device="cuda")

    # --- a1 ---
    def ntt(self, data: torch.Tensor, prime_idx, inverse: bool = False) -> torch.Tensor:
        """In place on data [n_polys][len(prime_idx)][N]."""
        pidx = (ctypes.c_int32 * len(prime_idx))(*prime_idx)
        n_polys = data.numel() // (len(prime_idx) * self.N)
        fn = lib().blb_intt if inverse else lib().blb_ntt
        _check(fn(self._h, _ptr(data), pidx, len(prime_idx), n_polys, _stream()))
        return data

    def intt(self, data, prime_idx):
        return self.ntt(data, prime_idx, inverse=True)

    # --- encode / decode ---
    def encode(self, slots: torch.Tensor, scale: float, level: int) -> torch.Tensor:
        """slots float64 [n_pts][N/2] (or [N/2]) on CUDA -> plaintexts int64 [n_pts][level+1][N]."""
        s = slots.to(device="cuda", dtype=torch.float64).contiguous()
        n_pts = 1 if s.dim() == 1 else s.shape[0]
        out = self.empty(n_pts, level + 1, self.N)
        _check(lib().blb_encode(self._h, _ptr(s), n_pts, float(scale), level, _ptr(out), _stream()))
        return out if s.dim() > 1 else out[0]

    def decode(self, pt: torch.Tensor, scale: float) -> torch.Tensor:
        level = pt.shape[0] - 1
        out = torch.empty(self.n, dtype=torch.float64, device="cuda")
        _check(lib().blb_decode(self._h, _ptr(pt.contiguous()), level, float(scale), _ptr(out), _stream()))
        return out


@dataclass
class Ciphertext:
    data: torch.Tensor  # int64 [2][level+1][N] CUDA
    level: int
    scale: float

    def c(self) -> _Ct:
        return _Ct(self.data.data_ptr(), self.level, 0, self.scale)

    @staticmethod
    def empty(params: Params, level: int, scale: float = 1.0) -> "Ciphertext":
        return Ciphertext(params.empty(2, level + 1, params.N), level, scale)


class Keys:
    def __init__(self, params: Params):
        self.params = params
        h = ctypes.c_void_p()
        _check(lib().blb_keys_create(params.handle, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.blb_keys_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def add(self, galois: int, swk: torch.Tensor):
        _check(lib().blb_keys_add(self._h, galois, _ptr(swk.contiguous()), _stream()))

    def has(self, galois: int) -> bool:
        return bool(lib().blb_keys_has(self._h, galois))


def keygen(params: Params, seed: bytes, rot_steps=(), relin: bool = False, want_secret: bool = True):
    keys = Keys(params)
    steps = (ctypes.c_int32 * max(1, len(rot_steps)))(*rot_steps)
    sk = params.empty(params.K + params.np_, params.N) if want_secret else None
    _check(lib().blb_keygen(params.handle, seed, steps, len(rot_steps), int(relin), keys.handle,
                            _ptr(sk) if sk is not None else None, _stream()))
    return keys, sk


def encrypt(params: Params, secret: torch.Tensor, pt: torch.Tensor, level: int, seed: bytes, ct_id: int,
            scale: float) -> Ciphertext:
    ct = Ciphertext.empty(params, level, scale)
    c = ct.c()
    _check(lib().blb_encrypt(params.handle, _ptr(secret), _ptr(pt.contiguous()), level, seed, ct_id, float(scale),
                             ctypes.byref(c), _stream()))
    return ct


def decrypt(params: Params, secret: torch.Tensor, ct: Ciphertext) -> torch.Tensor:
    out = params.empty(ct.level + 1, params.N)
    c = ct.c()
    _check(lib().blb_decrypt(params.handle, _ptr(secret), ctypes.byref(c), _ptr(out), _stream()))
    return out


def rotate(params: Params, keys: Keys, ct: Ciphertext, step: int, ws: torch.Tensor | None = None) -> Ciphertext:
    out = Ciphertext.empty(params, ct.level, ct.scale)
    ws = params.workspace(OP_ROTATE, ct.level) if ws is None else ws
    ci, co = ct.c(), out.c()
    _check(lib().blb_rotate(params.handle, keys.handle, ctypes.byref(ci), step, ctypes.byref(co), _ptr(ws),
                            ws.numel() * 8, _stream()))
    out.level, out.scale = co.level, co.scale
    return out


def rescale(params: Params, ct: Ciphertext, ws: torch.Tensor | None = None) -> Ciphertext:
    out = Ciphertext.empty(params, ct.level - 1)
    ws = params.workspace(OP_RESCALE, ct.level) if ws is None else ws
    ci, co = ct.c(), out.c()
    _check(lib().blb_rescale(params.handle, ctypes.byref(ci), ctypes.byref(co), _ptr(ws), ws.numel() * 8, _stream()))
    out.level, out.scale = co.level, co.scale
    return out


def mul_pt(params: Params, ct: Ciphertext, pt: torch.Tensor, pt_scale: float) -> Ciphertext:
    out = Ciphertext.empty(params, ct.level)
    ci, co = ct.c(), out.c()
    _check(lib().blb_mul_pt(params.handle, ctypes.byref(ci), _ptr(pt.contiguous()), float(pt_scale), ctypes.byref(co),
                            _stream()))
    out.level, out.scale = co.level, co.scale
    return out


def add(params: Params, a: Ciphertext, b: Ciphertext) -> Ciphertext:
    out = Ciphertext.empty(params, a.level)
    ca, cb, co = a.c(), b.c(), out.c()
    _check(lib().blb_add(params.handle, ctypes.byref(ca), ctypes.byref(cb), ctypes.byref(co), _stream()))
    out.level, out.scale = co.level, co.scale
    return out


def sub(params: Params, a: Ciphertext, b: Ciphertext) -> Ciphertext:
    out = Ciphertext.empty(params, a.level)
    ca, cb, co = a.c(), b.c(), out.c()
    _check(lib().blb_sub(params.handle, ctypes.byref(ca), ctypes.byref(cb), ctypes.byref(co), _stream()))
    out.level, out.scale = co.level, co.scale
    return out


def add_pt(params: Params, ct: Ciphertext, pt: torch.Tensor) -> Ciphertext:
    """ewadd_cp: (c0 + pt, c1); pt encoded at the ciphertext's scale and level."""
    out = Ciphertext.empty(params, ct.level)
    ci, co = ct.c(), out.c()
    _check(lib().blb_add_pt(params.handle, ctypes.byref(ci), _ptr(pt.contiguous()), ctypes.byref(co), _stream()))
    out.level, out.scale = co.level, co.scale
    return out


def drop_level(params: Params, ct: Ciphertext, level: int) -> Ciphertext:
    """Exact level drop (C9)."""
    out = Ciphertext.empty(params, level)
    ci, co = ct.c(), out.c()
    _check(lib().blb_drop_level(params.handle, ctypes.byref(ci), int(level), ctypes.byref(co), _stream()))
    out.level, out.scale = co.level, co.scale
    return out


def add_into(params: Params, a: Ciphertext, b: Ciphertext, out: Ciphertext) -> Ciphertext:
    ca, cb, co = a.c(), b.c(), out.c()
    _check(lib().blb_add(params.handle, ctypes.byref(ca), ctypes.byref(cb), ctypes.byref(co), _stream()))
    out.level, out.scale = co.level, co.scale
    return out


def ckks_to_mpc(params: Params, cts: list, mask_key: bytes, first_ct_id: int):
    """Server half of Alg. 1: returns (masked int64 [n][2][N], share int64 [n][N]), coefficient form mod q0."""
    n = len(cts)
    arr = (_Ct * n)(*[c.c() for c in cts])
    masked = params.empty(n, 2, params.N)
    share = params.empty(n, params.N)
    _check(lib().blb_ckks_to_mpc(params.handle, arr, n, mask_key, first_ct_id, _ptr(masked), _ptr(share), None, 0,
                                 _stream()))
    return masked, share


PK_ID = 1 << 55


def public_key(params: Params, secret: torch.Tensor, seed: bytes) -> Ciphertext:
    """The client's public key for S13: an encryption of zero at the top level, ciphertext id 2^55."""
    zero = params.empty(params.K, params.N).zero_()
    return encrypt(params, secret, zero, params.K - 1, seed, PK_ID, 1.0)


def ckks_to_mpc_rr(params: Params, pk: Ciphertext, cts: list, mask_key: bytes, rr_seed: bytes, first_ct_id: int,
                   flood_bits: int = 0):
    """S13 (reading C22): re-randomise with a fresh public-key encryption of zero (flooding noise of
    flood_bits), then the mask of Alg. 1.  Returns (masked int64 [n][2][N], share int64 [n][N])."""
    n = len(cts)
    arr = (_Ct * max(1, n))(*[c.c() for c in cts])
    masked = params.empty(n, 2, params.N)
    share = params.empty(n, params.N)
    nb = int(lib().blb_ckks_to_mpc_rr_workspace_bytes(params.handle, n))
    ws = torch.empty(max(1, nb // 8), dtype=torch.int64, device="cuda")
    pc = pk.c()
    _check(lib().blb_ckks_to_mpc_rr(params.handle, ctypes.byref(pc), arr, n, mask_key, rr_seed, first_ct_id,
                                    int(flood_bits), _ptr(masked), _ptr(share), _ptr(ws), ws.numel() * 8, _stream()))
    return masked, share


def share_to_rns(params: Params, x: torch.Tensor, w: int, sub: bool, level: int) -> torch.Tensor:
    """Row f3: a share over Z_{2^w} (int64 [N] CUDA, the u64 bit pattern) -> NTT residues [level+1][N]
    of x mod q_i (P0) or x - 2^w mod q_i (P1, sub)."""
    out = params.empty(level + 1, params.N)
    if x.dim() == 2:   # 128-bit shares [N][2] (w <= 128)
        _check(lib().blb_share_to_rns128(params.handle, _ptr(x.contiguous()), int(w), int(bool(sub)), level,
                                         _ptr(out), _stream()))
        return out
    _check(lib().blb_share_to_rns(params.handle, _ptr(x.contiguous()), int(w), int(bool(sub)), level, _ptr(out),
                                  _stream()))
    return out


def mpc_to_ckks(params: Params, ct: Ciphertext, x1: torch.Tensor, w: int) -> Ciphertext:
    """Row f3, server half of Alg. 2 line 4: ct (+) [tmp]_1^q, in place (c0 += NTT(x1 - 2^w mod q_i))."""
    ws = params.empty(ct.level + 1, params.N)
    c = ct.c()
    fn = lib().blb_mpc_to_ckks128 if x1.dim() == 2 else lib().blb_mpc_to_ckks
    _check(fn(params.handle, ctypes.byref(c), _ptr(x1.contiguous()), int(w), _ptr(ws), ws.numel() * 8, _stream()))
    return ct


def share_decode(params: Params, x: torch.Tensor, ft: int, s_out: int) -> torch.Tensor:
    """Row f3: local fixed-point Decode of a Z_{2^128} share (int64 [N][2] CUDA: lo, hi words) ->
    int64 [N/2][2] share of the real slots scaled by 2^-s_out (reading C18)."""
    y = torch.empty(params.N // 2, 2, dtype=torch.int64, device="cuda")
    ws = torch.empty(params.N * 6, dtype=torch.int64, device="cuda")
    _check(lib().blb_share_decode(params.handle, _ptr(x.contiguous()), int(ft), int(s_out), _ptr(y), _ptr(ws),
                                  ws.numel() * 8, _stream()))
    return y


def share_encode(params: Params, y: torch.Tensor, ft: int, s_out: int) -> torch.Tensor:
    """Row f3 (Alg. 2 line 1): local fixed-point Encode of a Z_{2^128} slot share (int64 [N/2][2] CUDA)
    -> int64 [N][2] share of the integer coefficients (reading C20)."""
    x = torch.empty(params.N, 2, dtype=torch.int64, device="cuda")
    ws = torch.empty(params.N * 6, dtype=torch.int64, device="cuda")
    _check(lib().blb_share_encode(params.handle, _ptr(y.contiguous()), int(ft), int(s_out), _ptr(x), _ptr(ws),
                                  ws.numel() * 8, _stream()))
    return x


def _f2_ws(params: Params, level: int) -> torch.Tensor:
    return torch.empty(int(lib().blb_f2_workspace_bytes(params.handle, level)) // 8 + 1, dtype=torch.int64,
                       device="cuda")


def mul_relin(params: Params, keys: Keys, a: Ciphertext, b: Ciphertext) -> Ciphertext:
    """ct x ct + relinearisation (row f2, C9); the caller rescales."""
    out = Ciphertext.empty(params, a.level)
    ws = _f2_ws(params, a.level)
    ca, cb, co = a.c(), b.c(), out.c()
    _check(lib().blb_mul_relin(params.handle, keys.handle, ctypes.byref(ca), ctypes.byref(cb), ctypes.byref(co),
                               _ptr(ws), ws.numel() * 8, _stream()))
    out.level, out.scale = co.level, co.scale
    return out


def mul_relin_batch(params: Params, keys: Keys, a: list, b: list, rescale: bool = True,
                    ws: torch.Tensor | None = None) -> list:
    """n pairs: tensor + relinearisation (+ rescale) in batched launches (row f2)."""
    n = len(a)
    if n == 0:
        return []
    lvl = a[0].level
    outs = [Ciphertext.empty(params, lvl - 1 if rescale else lvl) for _ in range(n)]
    nb = int(lib().blb_mul_relin_batch_workspace_bytes(params.handle, lvl, n))
    if ws is None or ws.numel() * 8 < nb:
        ws = torch.empty(nb // 8 + 1, dtype=torch.int64, device="cuda")
    ca = (_Ct * n)(*[c.c() for c in a])
    cb = (_Ct * n)(*[c.c() for c in b])
    co = (_Ct * n)(*[o.c() for o in outs])
    _check(lib().blb_mul_relin_batch(params.handle, keys.handle, ca, cb, n, int(bool(rescale)), co, _ptr(ws),
                                     ws.numel() * 8, _stream()))
    for o, c in zip(outs, co):
        o.level, o.scale = c.level, c.scale
    return outs


def mul_pt_rescale_batch(params: Params, cts: list, pts: list, pt_scales: list, ws: torch.Tensor | None = None) -> list:
    """n (ciphertext, plaintext) pairs: ct x pt then rescale, in batched launches (row f2)."""
    n = len(cts)
    if n == 0:
        return []
    lvl = cts[0].level
    outs = [Ciphertext.empty(params, lvl - 1) for _ in range(n)]
    nb = int(lib().blb_mul_pt_rescale_batch_workspace_bytes(params.handle, lvl, n))
    if ws is None or ws.numel() * 8 < nb:
        ws = torch.empty(nb // 8 + 1, dtype=torch.int64, device="cuda")
    ci = (_Ct * n)(*[c.c() for c in cts])
    co = (_Ct * n)(*[o.c() for o in outs])
    pp = (ctypes.c_void_p * n)(*[p.data_ptr() for p in pts])
    ps = (ctypes.c_double * n)(*[float(s) for s in pt_scales])
    _check(lib().blb_mul_pt_rescale_batch(params.handle, ci, pp, ps, n, co, _ptr(ws), ws.numel() * 8, _stream()))
    for o, c in zip(outs, co):
        o.level, o.scale = c.level, c.scale
    return outs


def rotate_sum(params: Params, keys: Keys, ct: Ciphertext, L: int, D: int, broadcast: bool = False) -> Ciphertext:
    """Rotate-and-sum: log2 D rotations, fused form (no mask)."""
    out = Ciphertext.empty(params, ct.level)
    ws = _f2_ws(params, ct.level)
    ci, co = ct.c(), out.c()
    fn = lib().blb_broadcast if broadcast else lib().blb_rotate_sum
    _check(fn(params.handle, keys.handle, ctypes.byref(ci), L, D, ctypes.byref(co), _ptr(ws), ws.numel() * 8,
              _stream()))
    out.level, out.scale = co.level, co.scale
    return out


def mhp_column_map(d: int, heads: int, L: int, log_n: int) -> list[int]:
    n = ctypes.c_int(0)
    _check(lib().blb_mhp_column_map(d, heads, L, log_n, None, ctypes.byref(n)))
    buf = (ctypes.c_int32 * n.value)()
    _check(lib().blb_mhp_column_map(d, heads, L, log_n, buf, ctypes.byref(n)))
    return [int(x) for x in buf]


class MatmulPlan:
    """blb_matmul_plan_create (C11 spatial / C12 diagonal ct-pt MatMul with BSGS)."""

    def __init__(self, params: Params, L: int, w_rows: int, w_cols: int, packing: int = PACK_SPATIAL, heads: int = 1,
                 col_map=None, bsgs_B: int = 16, level: int | None = None, window: tuple | None = None):
        """window = (i_first, i_count): the plan restricted to a baby-step window (multi-GPU, DESIGN
        section 8); None = the whole plan."""
        self.params = params
        self.window = window
        self.level = params.K - 1 if level is None else level
        self.w_shape = (w_rows, w_cols)
        cm = None
        d_out = w_cols
        if col_map is not None:
            cm = (ctypes.c_int32 * len(col_map))(*col_map)
            d_out = len(col_map)
        h = ctypes.c_void_p()
        if window is None:
            _check(lib().blb_matmul_plan_create(params.handle, L, w_rows, w_cols, packing, heads, cm, d_out, bsgs_B,
                                                self.level, ctypes.byref(h)))
        else:
            _check(lib().blb_matmul_plan_create_window(params.handle, L, w_rows, w_cols, packing, heads, cm, d_out,
                                                       bsgs_B, self.level, int(window[0]), int(window[1]),
                                                       ctypes.byref(h)))
        self._h = h
        vals = [ctypes.c_int() for _ in range(7)]
        _check(lib().blb_matmul_plan_info(h, *[ctypes.byref(v) for v in vals]))
        self.n_in, self.n_out, self.n_pt, self.n_baby, self.n_giant, self.B, self.G = [v.value for v in vals]

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.blb_matmul_plan_destroy(self._h)
            self._h = None

    @property
    def n_rotations(self) -> int:
        return self.n_baby + self.n_giant

    def rotation_steps(self) -> list[int]:
        n = ctypes.c_int(0)
        _check(lib().blb_matmul_plan_rotations(self._h, None, ctypes.byref(n)))
        buf = (ctypes.c_int32 * max(1, n.value))()
        _check(lib().blb_matmul_plan_rotations(self._h, buf, ctypes.byref(n)))
        return [int(buf[i]) for i in range(n.value)]

    def pt_count(self, out_first: int = 0, out_count: int | None = None) -> int:
        out_count = self.n_out - out_first if out_count is None else out_count
        n = ctypes.c_int(0)
        _check(lib().blb_matmul_pt_count(self._h, out_first, out_count, ctypes.byref(n)))
        return n.value

    def encode_weights(self, W, out_first: int = 0, out_count: int | None = None,
                       out: torch.Tensor | None = None) -> torch.Tensor:
        """W: host float64 array or a device float64 tensor (per-layer re-encode); out: reuse a buffer."""
        out_count = self.n_out - out_first if out_count is None else out_count
        if isinstance(W, torch.Tensor):
            assert W.dtype == torch.float64 and W.is_contiguous() and tuple(W.shape) == self.w_shape
            wptr = ctypes.c_void_p(W.data_ptr())
        else:
            W = np.ascontiguousarray(W, dtype=np.float64)
            assert W.shape == self.w_shape
            wptr = W.ctypes.data_as(ctypes.c_void_p)
        nbytes = ctypes.c_size_t(0)
        _check(lib().blb_matmul_pt_bytes(self._h, out_first, out_count, ctypes.byref(nbytes)))
        # opaque width-packed blocked layout (include/blb.h): int64 words, 16-byte aligned
        n = max(1, (nbytes.value + 7) // 8)
        pts = torch.empty(n, dtype=torch.int64, device="cuda") if out is None else out
        assert pts.numel() >= n
        _check(lib().blb_matmul_encode_weights(self._h, wptr, out_first, out_count, _ptr(pts), _stream()))
        return pts

    def _wptr(self, W):
        if isinstance(W, torch.Tensor):
            assert W.dtype == torch.float64 and W.is_contiguous() and tuple(W.shape) == self.w_shape
            return W, ctypes.c_void_p(W.data_ptr())
        W = np.ascontiguousarray(W, dtype=np.float64)
        assert W.shape == self.w_shape
        return W, W.ctypes.data_as(ctypes.c_void_p)

    def encode_coeffs(self, W, out_first: int = 0, out_count: int | None = None,
                      out: torch.Tensor | None = None) -> torch.Tensor:
        """Compact prime-independent weights of the slice (5-byte coefficients, opaque uint8 buffer)."""
        out_count = self.n_out - out_first if out_count is None else out_count
        W, wptr = self._wptr(W)
        nbytes = ctypes.c_size_t(0)
        _check(lib().blb_matmul_coeff_bytes(self._h, out_first, out_count, ctypes.byref(nbytes)))
        coef = torch.empty(max(1, nbytes.value), dtype=torch.uint8, device="cuda") if out is None else out
        assert coef.numel() >= nbytes.value
        _check(lib().blb_matmul_encode_coeffs(self._h, wptr, out_first, out_count, _ptr(coef), _stream()))
        return coef

    def coeffs_to_pts(self, coef: torch.Tensor, out_first: int = 0, out_count: int | None = None,
                      out: torch.Tensor | None = None) -> torch.Tensor:
        """Expand encode_coeffs output into the plaintext buffer encode_weights would produce (no sync)."""
        out_count = self.n_out - out_first if out_count is None else out_count
        nbytes = ctypes.c_size_t(0)
        _check(lib().blb_matmul_pt_bytes(self._h, out_first, out_count, ctypes.byref(nbytes)))
        n = max(1, (nbytes.value + 7) // 8)
        pts = torch.empty(n, dtype=torch.int64, device="cuda") if out is None else out
        assert pts.numel() >= n
        _check(lib().blb_matmul_coeffs_to_pts(self._h, _ptr(coef), out_first, out_count, _ptr(pts), _stream()))
        return pts

    def workspace_bytes(self, out_count: int | None = None) -> int:
        out_count = self.n_out if out_count is None else out_count
        return int(lib().blb_matmul_workspace_bytes(self._h, out_count))

    def workspace(self, out_count: int | None = None) -> torch.Tensor:
        nbytes = self.workspace_bytes(out_count)
        return torch.empty(nbytes // 8 + 1, dtype=torch.int64, device="cuda")

    def __call__(self, keys: Keys, cts: list, pts: torch.Tensor, out_first: int = 0, out_count: int | None = None,
                 ws: torch.Tensor | None = None, outs: list | None = None) -> list:
        out_count = self.n_out - out_first if out_count is None else out_count
        ws = self.workspace(out_count) if ws is None else ws
        if outs is None:
            outs = [Ciphertext.empty(self.params, self.level - 1) for _ in range(out_count)]
        cin = (_Ct * len(cts))(*[c.c() for c in cts])
        cout = (_Ct * max(1, out_count))(*[o.c() for o in outs])
        _check(lib().blb_ct_pt_matmul(self._h, keys.handle, cin, len(cts), _ptr(pts), out_first, out_count, cout,
                                      _ptr(ws), ws.numel() * 8, _stream()))
        for o, c in zip(outs, cout):
            o.level, o.scale = c.level, c.scale
        return outs

    def batch(self, keys: Keys, cts_sets: list, pts: torch.Tensor, out_first: int = 0, out_count: int | None = None,
              ws: torch.Tensor | None = None) -> list:
        """blb_ct_pt_matmul_batch: several input sets against the same plaintexts (one weight-stationary
        MAC); -> one list of outputs per set."""
        out_count = self.n_out - out_first if out_count is None else out_count
        nb = len(cts_sets)
        n_in = len(cts_sets[0])
        assert all(len(c) == n_in for c in cts_sets)
        per = self.workspace_bytes(out_count)
        ws = torch.empty(nb * per // 8 + 1, dtype=torch.int64, device="cuda") if ws is None else ws
        outs = [[Ciphertext.empty(self.params, self.level - 1) for _ in range(out_count)] for _ in range(nb)]
        flat_in = [c for cs in cts_sets for c in cs]
        flat_out = [o for os_ in outs for o in os_]
        cin = (_Ct * len(flat_in))(*[c.c() for c in flat_in])
        cout = (_Ct * max(1, len(flat_out)))(*[o.c() for o in flat_out])
        _check(lib().blb_ct_pt_matmul_batch(self._h, keys.handle, cin, n_in, nb, _ptr(pts), out_first, out_count, cout,
                                            _ptr(ws), ws.numel() * 8, _stream()))
        for o, c in zip(flat_out, cout):
            o.level, o.scale = c.level, c.scale
        return outs

    def acc_numel(self, n_out: int | None = None) -> int:
        """u64 words of the MAC accumulators of n_out outputs: [n_out][G][2][level+1][N]."""
        n_out = self.n_out if n_out is None else n_out
        return n_out * self.G * 2 * (self.level + 1) * self.params.N

    def acc(self, keys: Keys, cts: list, pts: torch.Tensor, acc_out: torch.Tensor | None = None,
            ws: torch.Tensor | None = None) -> torch.Tensor:
        """blb_ct_pt_matmul_acc: baby steps + MAC of this plan's window for every output."""
        ws = self.workspace(0) if ws is None else ws
        acc_out = torch.empty(self.acc_numel(), dtype=torch.int64, device="cuda") if acc_out is None else acc_out
        assert acc_out.numel() >= self.acc_numel()
        cin = (_Ct * len(cts))(*[c.c() for c in cts])
        _check(lib().blb_ct_pt_matmul_acc(self._h, keys.handle, cin, len(cts), _ptr(pts), _ptr(acc_out), _ptr(ws),
                                          ws.numel() * 8, _stream()))
        return acc_out

    def finish(self, keys: Keys, acc_in: torch.Tensor, out_first: int, out_count: int, scale: float,
               ws: torch.Tensor | None = None, outs: list | None = None) -> list:
        """blb_ct_pt_matmul_finish: giant steps + ModDown/rescale of outputs [out_first, +out_count) from
        the cross-rank SUM of their accumulators."""
        ws = self.workspace(out_count) if ws is None else ws
        if outs is None:
            outs = [Ciphertext.empty(self.params, self.level - 1) for _ in range(out_count)]
        cout = (_Ct * max(1, out_count))(*[o.c() for o in outs])
        _check(lib().blb_ct_pt_matmul_finish(self._h, keys.handle, _ptr(acc_in), out_first, out_count, float(scale),
                                             cout, _ptr(ws), ws.numel() * 8, _stream()))
        for o, c in zip(outs, cout):
            o.level, o.scale = c.level, c.scale
        return outs


class QKPlan:
    """blb_qk_plan_create: ct-ct MatMul Q_h K_h^T for all heads (row a7, reading C13)."""

    def __init__(self, params: Params, L: int, heads: int, d_h: int, bsgs_B: int = 0, level: int | None = None,
                 window: tuple | None = None):
        """window = (i_first, i_count): the plan restricted to a baby-index window (multi-GPU)."""
        self.params = params
        self.level = params.K - 2 if level is None else level
        self.window = window
        h = ctypes.c_void_p()
        if window is None:
            _check(lib().blb_qk_plan_create(params.handle, L, heads, d_h, bsgs_B, self.level, ctypes.byref(h)))
        else:
            _check(lib().blb_qk_plan_create_window(params.handle, L, heads, d_h, bsgs_B, self.level, int(window[0]),
                                                   int(window[1]), ctypes.byref(h)))
        self._h = h
        vals = [ctypes.c_int() for _ in range(7)]
        _check(lib().blb_qk_plan_info(h, *[ctypes.byref(v) for v in vals]))
        self.J, self.n_out, self.g, self.B, self.G, self.n_rotations, self.n_masks = [v.value for v in vals]

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.blb_qk_plan_destroy(self._h)
            self._h = None

    def rotation_steps(self) -> list[int]:
        n = ctypes.c_int(0)
        _check(lib().blb_qk_plan_rotations(self._h, None, ctypes.byref(n)))
        buf = (ctypes.c_int32 * max(1, n.value))()
        _check(lib().blb_qk_plan_rotations(self._h, buf, ctypes.byref(n)))
        return [int(buf[i]) for i in range(n.value)]

    def encode_masks(self) -> torch.Tensor:
        nbytes = int(lib().blb_qk_mask_bytes(self._h))
        masks = torch.empty(nbytes // 8, dtype=torch.int64, device="cuda")
        _check(lib().blb_qk_encode_masks(self._h, _ptr(masks), _stream()))
        return masks

    def workspace_bytes(self) -> int:
        return int(lib().blb_qk_workspace_bytes(self._h))

    def __call__(self, keys: Keys, Q: list, K: list, masks: torch.Tensor, ws: torch.Tensor | None = None,
                 outs: list | None = None) -> list:
        ws = torch.empty(self.workspace_bytes() // 8 + 1, dtype=torch.int64, device="cuda") if ws is None else ws
        if outs is None:
            outs = [Ciphertext.empty(self.params, self.level - 3) for _ in range(self.n_out)]
        cq = (_Ct * len(Q))(*[c.c() for c in Q])
        ck = (_Ct * len(K))(*[c.c() for c in K])
        co = (_Ct * self.n_out)(*[o.c() for o in outs])
        _check(lib().blb_ct_ct_qk(self._h, keys.handle, cq, ck, len(Q), _ptr(masks), co, _ptr(ws), ws.numel() * 8,
                                  _stream()))
        for o, c in zip(outs, co):
            o.level, o.scale = c.level, c.scale
        return outs

    def acc_numel(self) -> int:
        return int(lib().blb_qk_acc_bytes(self._h)) // 8

    def acc_range(self, out_first: int, out_count: int) -> tuple:
        """Accumulator slots (first, count) read by outputs [out_first, out_first + out_count)."""
        a, b = ctypes.c_int(), ctypes.c_int()
        _check(lib().blb_qk_acc_range(self._h, out_first, out_count, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def acc(self, keys: Keys, Q: list, K: list, masks: torch.Tensor, acc_out: torch.Tensor | None = None,
            ws: torch.Tensor | None = None) -> torch.Tensor:
        """blb_ct_ct_qk_acc: this window's step-3 accumulators (before ModDown + rescale)."""
        ws = torch.empty(self.workspace_bytes() // 8 + 1, dtype=torch.int64, device="cuda") if ws is None else ws
        acc_out = torch.empty(self.acc_numel(), dtype=torch.int64, device="cuda") if acc_out is None else acc_out
        cq = (_Ct * len(Q))(*[c.c() for c in Q])
        ck = (_Ct * len(K))(*[c.c() for c in K])
        _check(lib().blb_ct_ct_qk_acc(self._h, keys.handle, cq, ck, len(Q), _ptr(masks), _ptr(acc_out), _ptr(ws),
                                      ws.numel() * 8, _stream()))
        return acc_out

    def finish(self, keys: Keys, acc_in: torch.Tensor, out_first: int, out_count: int, scale_q: float, scale_k: float,
               ws: torch.Tensor | None = None, outs: list | None = None) -> list:
        """blb_ct_ct_qk_finish: outputs [out_first, +out_count) from the summed accumulator slots
        acc_range(out_first, out_count) (acc_in starts at the first of them)."""
        ws = torch.empty(self.workspace_bytes() // 8 + 1, dtype=torch.int64, device="cuda") if ws is None else ws
        if outs is None:
            outs = [Ciphertext.empty(self.params, self.level - 3) for _ in range(out_count)]
        co = (_Ct * max(1, out_count))(*[o.c() for o in outs])
        _check(lib().blb_ct_ct_qk_finish(self._h, keys.handle, _ptr(acc_in), out_first, out_count, float(scale_q),
                                         float(scale_k), co, _ptr(ws), ws.numel() * 8, _stream()))
        for o, c in zip(outs, co):
            o.level, o.scale = c.level, c.scale
        return outs
