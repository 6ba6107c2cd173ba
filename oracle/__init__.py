"""BLB CKKS oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU statement of the server-side CKKS hot path
of BLB (arXiv 2508.19525): NTT, encode, keys, encrypt/decrypt, hoisted
rotation with hybrid key switching (ModUp/ModDown), rescale, ct-pt products
and the CKKS->MPC mask.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_2508_19525_b200`` (the product) and
never imports it.

Arithmetic lives in ``blb_oracle.c`` (exact u128 modular arithmetic,
__float128 encode); this module only marshals numpy arrays and states the
protocol-level order of operations.  Citations: ``P:n`` = PAPER.md line n;
``C<k>`` = DESIGN.md reading k.

Parity status: every function here is pinned by tests/test_oracle_*.py
(closed forms, brute force, exact big-integer invariants, RFC/KAT vectors);
see DESIGN.md "Oracle pins".
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

TAG_SECRET, TAG_KEY_A, TAG_KEY_E, TAG_ENC_A, TAG_ENC_E, TAG_MASK = 1, 2, 3, 4, 5, 6
TAG_RR_V, TAG_RR_E0, TAG_RR_E1 = 7, 8, 9     # S13 re-randomisation draws (reading C22)
PK_ID = 1 << 55                               # ciphertext id of the public key (an encryption of zero)


def build(force: bool = False) -> str:
    """Compile blb_oracle.c -> liboracle.so (gcc, OpenMP, libquadmath)."""
    src = os.path.join(_HERE, "blb_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        import subprocess
        tmp = _SO + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, src, "-lquadmath"])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        L.orc_ctx_new.restype = ctypes.c_void_p
        L.orc_ctx_new.argtypes = [ctypes.c_int, u64p, ctypes.c_int, u64p, ctypes.c_int, ctypes.c_int,
                                  ctypes.POINTER(ctypes.c_int)]
        L.orc_ctx_free.argtypes = [ctypes.c_void_p]
        L.orc_ctx_alpha.argtypes = [ctypes.c_void_p]
        L.orc_ctx_psi.restype = ctypes.c_uint64
        L.orc_ctx_psi.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.orc_min_psi.restype = ctypes.c_uint64
        L.orc_min_psi.argtypes = [ctypes.c_uint64, ctypes.c_int]
        L.orc_is_prime.argtypes = [ctypes.c_uint64]
        L.orc_prime_chain.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int, u64p]
        L.orc_mulmod.restype = ctypes.c_uint64
        L.orc_mulmod.argtypes = [ctypes.c_uint64] * 3
        L.orc_encode_coeffs.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p]
        L.orc_encode.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_void_p]
        L.orc_encode_direct.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p,
                                        ctypes.c_void_p]
        L.orc_quad_to_str.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int]
        for name in ("orc_ntt", "orc_intt"):
            getattr(L, name).argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.orc_negacyclic_schoolbook.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_uint64] * 2
        L.orc_automorphism_ntt.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                           ctypes.c_int]
        L.orc_automorphism_coef.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                            ctypes.c_uint64]
        L.orc_chacha20_block.argtypes = [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_char_p, ctypes.c_void_p]
        L.orc_draw128.argtypes = [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                  ctypes.c_void_p]
        for name in ("orc_sample_uniform",):
            getattr(L, name).argtypes = [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_uint64, ctypes.c_void_p]
        for name in ("orc_sample_ternary", "orc_sample_cbd"):
            getattr(L, name).argtypes = [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_void_p]
        L.orc_secret.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_gen_swk.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_uint64, ctypes.c_void_p]
        L.orc_encrypt.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p]
        L.orc_decrypt.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                  ctypes.c_void_p]
        L.orc_fastbconv.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64,
                                    ctypes.c_void_p, ctypes.c_uint64]
        L.orc_modup.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        L.orc_moddown.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        L.orc_ks_inner.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                   ctypes.c_uint64, ctypes.c_void_p]
        L.orc_rotate.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                 ctypes.c_uint64, ctypes.c_void_p]
        L.orc_tensor.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                 ctypes.c_void_p]
        L.orc_relinearize.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                      ctypes.c_void_p]
        L.orc_mul_pt.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                 ctypes.c_void_p]
        L.orc_add.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                              ctypes.c_void_p]
        L.orc_rescale.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.orc_mask.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_char_p, ctypes.c_uint64,
                               ctypes.c_void_p, ctypes.c_void_p]
        L.orc_rotate_ext.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_uint64, ctypes.c_void_p]
        for name in ("orc_mul_pt_idx", "orc_add_idx"):
            getattr(L, name).argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.orc_encode_ext.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_int,
                                     ctypes.c_void_p]
        L.orc_moddown_rescale.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        L.orc_share_decode.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.orc_share_encode.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.orc_share_to_rns128.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_void_p]
        L.orc_share_to_rns.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_void_p]
        L.orc_relinearize_ext.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                          ctypes.c_void_p]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


# ---------------------------------------------------------------------------
# parameters (C1)
# ---------------------------------------------------------------------------
def prime_chain(log_n: int, bits: list[int]) -> list[int]:
    """C1 prime-list rule: largest unused prime < 2^b, == 1 mod 2N, in order."""
    out = (ctypes.c_uint64 * len(bits))()
    b = (ctypes.c_int * len(bits))(*bits)
    st = lib().orc_prime_chain(log_n, b, len(bits), out)
    if st != 0:
        raise ValueError("prime chain failed: %d" % st)
    return [int(x) for x in out]


def min_psi(q: int, log_n: int) -> int:
    return int(lib().orc_min_psi(q, log_n))


class ParamError(ValueError):
    pass


class Ctx:
    """Oracle parameter context: N = 2^log_n, chain q (K primes), special p, dnum (C1)."""

    def __init__(self, log_n: int, q: list[int], p: list[int], dnum: int):
        self.log_n, self.N, self.n = log_n, 1 << log_n, 1 << (log_n - 1)
        self.q, self.p = [int(x) for x in q], [int(x) for x in p]
        self.K, self.np_ = len(q), len(p)
        self.mods = self.q + self.p
        self.dnum = dnum
        qa = (ctypes.c_uint64 * self.K)(*self.q)
        pa = (ctypes.c_uint64 * self.np_)(*self.p)
        st = ctypes.c_int(0)
        self._h = lib().orc_ctx_new(log_n, qa, self.K, pa, self.np_, dnum, ctypes.byref(st))
        if not self._h:
            raise ParamError("orc_ctx_new status %d" % st.value)
        self.alpha = lib().orc_ctx_alpha(self._h)
        self.psi = [int(lib().orc_ctx_psi(self._h, i)) for i in range(self.K + self.np_)]

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_ctx_free(self._h)
            self._h = None

    def beta(self, level: int) -> int:
        return -(-(level + 1) // self.alpha)

    @property
    def beta_top(self) -> int:
        return -(-self.K // self.alpha)

    def P(self) -> int:
        r = 1
        for x in self.p:
            r *= x
        return r

    # ---- NTT (C2) ----
    def ntt(self, a: np.ndarray, pidx) -> np.ndarray:
        a = _u64(a).copy()
        pa = (ctypes.c_int * len(pidx))(*pidx)
        lib().orc_ntt(self._h, _p(a), pa, len(pidx))
        return a

    def intt(self, a: np.ndarray, pidx) -> np.ndarray:
        a = _u64(a).copy()
        pa = (ctypes.c_int * len(pidx))(*pidx)
        lib().orc_intt(self._h, _p(a), pa, len(pidx))
        return a

    def automorphism_ntt(self, a: np.ndarray, g: int) -> np.ndarray:
        a = _u64(a)
        out = np.empty_like(a)
        limbs = a.size // self.N
        lib().orc_automorphism_ntt(self._h, _p(a), _p(out), g, limbs)
        return out

    def galois(self, step: int) -> int:
        """Left rotation by `step` slots <-> X -> X^(5^step mod 2N) (C3)."""
        return pow(5, step % self.n, 2 * self.N)


def schoolbook(a, b, q: int) -> np.ndarray:
    a, b = _u64(a), _u64(b)
    out = np.empty_like(a)
    lib().orc_negacyclic_schoolbook(_p(a), _p(b), _p(out), a.size, q)
    return out


def automorphism_coef(a, g: int, q: int) -> np.ndarray:
    a = _u64(a)
    out = np.empty_like(a)
    lib().orc_automorphism_coef(a.size, _p(a), _p(out), g, q)
    return out


def fastbconv(src: np.ndarray, cm: list[int], dm: int) -> np.ndarray:
    src = _u64(src)
    N = src.shape[-1]
    out = np.empty(N, dtype=np.uint64)
    cma = _u64(cm)
    lib().orc_fastbconv(_p(src), _p(cma), len(cm), dm, _p(out), N)
    return out


# ---------------------------------------------------------------------------
# randomness (C4)
# ---------------------------------------------------------------------------
def chacha20_block(key: bytes, counter: int, nonce: bytes) -> bytes:
    out = (ctypes.c_uint8 * 64)()
    lib().orc_chacha20_block(key, counter, nonce, out)
    return bytes(out)


def draw128(key: bytes, tag: int, objid: int, x: int) -> int:
    out = np.zeros(2, dtype=np.uint64)
    lib().orc_draw128(key, tag, objid, x, _p(out))
    return int(out[0]) | (int(out[1]) << 64)


def sample_uniform(key: bytes, tag: int, objid: int, q: int, N: int) -> np.ndarray:
    out = np.empty(N, dtype=np.uint64)
    lib().orc_sample_uniform(key, tag, objid, q, N, _p(out))
    return out


def sample_ternary(key: bytes, tag: int, objid: int, N: int) -> np.ndarray:
    out = np.empty(N, dtype=np.int64)
    lib().orc_sample_ternary(key, tag, objid, N, _p(out))
    return out


def sample_cbd(key: bytes, tag: int, objid: int, N: int) -> np.ndarray:
    out = np.empty(N, dtype=np.int64)
    lib().orc_sample_cbd(key, tag, objid, N, _p(out))
    return out


# ---------------------------------------------------------------------------
# encode / decode (C3)
# ---------------------------------------------------------------------------
class EncodeOverflow(ValueError):
    pass


def encode_coeffs(ctx: Ctx, z, scale: float) -> np.ndarray:
    """round(scale * pi^{-1}(z)) as int64 coefficients (correctly rounded, ties-to-even)."""
    z = np.ascontiguousarray(z, dtype=np.float64)
    assert z.shape == (ctx.n,)
    out = np.empty(ctx.N, dtype=np.int64)
    if lib().orc_encode_coeffs(ctx._h, _p(z), float(scale), _p(out)) != 0:
        raise EncodeOverflow("encode magnitude >= 2^62")
    return out


def encode(ctx: Ctx, z, scale: float, level: int) -> np.ndarray:
    """Plaintext in NTT form over q_0..q_level: [level+1][N]."""
    z = np.ascontiguousarray(z, dtype=np.float64)
    assert z.shape == (ctx.n,)
    out = np.empty((level + 1, ctx.N), dtype=np.uint64)
    if lib().orc_encode(ctx._h, _p(z), float(scale), level, _p(out)) != 0:
        raise EncodeOverflow("encode magnitude >= 2^62")
    return out


def encode_direct(ctx: Ctx, z, scale: float):
    """Direct O(N n) evaluation of the same definition (pins only): (exact quad strings, rounded)."""
    z = np.ascontiguousarray(z, dtype=np.float64)
    coef = np.empty(ctx.N, dtype=np.int64)
    lib().orc_encode_direct(ctx._h, _p(z), float(scale), None, _p(coef))
    return coef


def crt_centered(ctx: Ctx, limbs_coef: np.ndarray) -> list[int]:
    """Exact centred CRT lift over q_0..q_{k-1} of coefficient-form residues [k][N]."""
    k = limbs_coef.shape[0]
    mods = ctx.q[:k]
    Q = 1
    for m in mods:
        Q *= m
    terms = []
    for i, m in enumerate(mods):
        qh = Q // m
        terms.append((qh * pow(qh % m, -1, m)) % Q)
    out = []
    cols = [limbs_coef[i].tolist() for i in range(k)]
    for x in range(limbs_coef.shape[1]):
        v = 0
        for i in range(k):
            v += cols[i][x] * terms[i]
        v %= Q
        if v > Q // 2:
            v -= Q
        out.append(v)
    return out


def decode_coeffs(ctx: Ctx, coef: list[int] | np.ndarray, scale: float) -> np.ndarray:
    """z_j = Re(sum_k m_k zeta^{k 5^j}) / scale  (pi of Eq. eq:ckks_encode, real slots).

    Evaluated as sum_k (m_k zeta^k) omega^{k t} with 2t+1 = 5^j mod 2N, i.e. one
    numpy inverse FFT (a library step); pinned against the direct sum in tests."""
    N, n = ctx.N, ctx.n
    m = np.array([float(v) for v in coef], dtype=np.float64)
    k = np.arange(N)
    zeta_k = np.exp(1j * np.pi * k / N)
    S = np.fft.ifft(m * zeta_k) * N
    t = np.array([(pow(5, j, 2 * N) - 1) // 2 for j in range(n)])
    return S[t].real / scale


def decode(ctx: Ctx, pt: np.ndarray, scale: float) -> np.ndarray:
    k = pt.shape[0]
    coef = ctx.intt(pt, list(range(k)))
    return decode_coeffs(ctx, crt_centered(ctx, coef), scale)


# ---------------------------------------------------------------------------
# ciphertexts, keys (C5, C6)
# ---------------------------------------------------------------------------
@dataclass
class Ct:
    data: np.ndarray  # [2][level+1][N] uint64, NTT domain
    level: int
    scale: float

    def copy(self) -> "Ct":
        return Ct(self.data.copy(), self.level, self.scale)


@dataclass
class Keys:
    s_coef: np.ndarray
    s_ntt: np.ndarray                       # [K+np][N]
    rot: dict = field(default_factory=dict)  # galois element -> [beta_top][2][K+np][N]
    rlk: np.ndarray | None = None


def secret(ctx: Ctx, key: bytes):
    s_coef = np.empty(ctx.N, dtype=np.int64)
    s_ntt = np.empty((ctx.K + ctx.np_, ctx.N), dtype=np.uint64)
    lib().orc_secret(ctx._h, key, _p(s_coef), _p(s_ntt))
    return s_coef, s_ntt


def gen_swk(ctx: Ctx, key: bytes, s_ntt: np.ndarray, target_ntt: np.ndarray, key_id: int) -> np.ndarray:
    out = np.empty((ctx.beta_top, 2, ctx.K + ctx.np_, ctx.N), dtype=np.uint64)
    lib().orc_gen_swk(ctx._h, key, _p(_u64(s_ntt)), _p(_u64(target_ntt)), key_id, _p(out))
    return out


def keygen(ctx: Ctx, key: bytes, rot_steps=(), relin: bool = False) -> Keys:
    """Client-side key generation (C5).  Rotation key for step r targets sigma_g(s),
    g = 5^r mod 2N, ChaCha key id = g; the relinearisation key targets s^2, id 0."""
    s_coef, s_ntt = secret(ctx, key)
    keys = Keys(s_coef, s_ntt)
    for r in rot_steps:
        g = ctx.galois(r)
        if g in keys.rot or g == 1:
            continue
        keys.rot[g] = gen_swk(ctx, key, s_ntt, ctx.automorphism_ntt(s_ntt, g), g)
    if relin:
        s2 = np.empty_like(s_ntt)
        for i, m in enumerate(ctx.mods):
            s2[i] = np.array([(int(a) * int(a)) % m for a in s_ntt[i].tolist()], dtype=np.uint64)
        keys.rlk = gen_swk(ctx, key, s_ntt, s2, 0)
    return keys


def encrypt(ctx: Ctx, key: bytes, s_ntt: np.ndarray, pt: np.ndarray, level: int, ct_id: int, scale: float) -> Ct:
    out = np.empty((2, level + 1, ctx.N), dtype=np.uint64)
    lib().orc_encrypt(ctx._h, key, _p(_u64(s_ntt)), _p(_u64(pt[: level + 1])), level, ct_id, _p(out))
    return Ct(out, level, scale)


def decrypt(ctx: Ctx, s_ntt: np.ndarray, ct: Ct) -> np.ndarray:
    out = np.empty((ct.level + 1, ctx.N), dtype=np.uint64)
    lib().orc_decrypt(ctx._h, _p(_u64(s_ntt)), _p(_u64(ct.data)), ct.level, _p(out))
    return out


# ---------------------------------------------------------------------------
# key switching (C7, C8), products (C9), rescale (C10), mask (C14)
# ---------------------------------------------------------------------------
def modup(ctx: Ctx, d: np.ndarray, level: int) -> np.ndarray:
    E = level + 1 + ctx.np_
    out = np.empty((ctx.beta(level), E, ctx.N), dtype=np.uint64)
    lib().orc_modup(ctx._h, _p(_u64(d)), level, _p(out))
    return out


def moddown(ctx: Ctx, y: np.ndarray, level: int) -> np.ndarray:
    out = np.empty((level + 1, ctx.N), dtype=np.uint64)
    lib().orc_moddown(ctx._h, _p(_u64(y)), level, _p(out))
    return out


def rotate(ctx: Ctx, ct: Ct, keys: Keys, step: int) -> Ct:
    """Left rotation by `step` slots, hoisted form (C8)."""
    g = ctx.galois(step)
    if g == 1:
        return ct.copy()
    if g not in keys.rot:
        raise KeyError("missing rotation key for step %d" % step)
    out = np.empty_like(ct.data)
    lib().orc_rotate(ctx._h, _p(_u64(ct.data)), ct.level, _p(keys.rot[g]), g, _p(out))
    return Ct(out, ct.level, ct.scale)


def mul_pt(ctx: Ctx, ct: Ct, pt: np.ndarray, pt_scale: float) -> Ct:
    out = np.empty_like(ct.data)
    lib().orc_mul_pt(ctx._h, _p(_u64(ct.data)), _p(_u64(pt[: ct.level + 1])), ct.level, _p(out))
    return Ct(out, ct.level, ct.scale * pt_scale)


def add(ctx: Ctx, a: Ct, b: Ct) -> Ct:
    assert a.level == b.level and a.data.shape == b.data.shape
    out = np.empty_like(a.data)
    lib().orc_add(ctx._h, _p(_u64(a.data)), _p(_u64(b.data)), a.level, a.data.shape[0], _p(out))
    return Ct(out, a.level, a.scale)


def tensor(ctx: Ctx, a: Ct, b: Ct) -> Ct:
    out = np.empty((3, a.level + 1, ctx.N), dtype=np.uint64)
    lib().orc_tensor(ctx._h, _p(_u64(a.data)), _p(_u64(b.data)), a.level, _p(out))
    return Ct(out, a.level, a.scale * b.scale)


def relinearize(ctx: Ctx, d: Ct, keys: Keys) -> Ct:
    out = np.empty((2, d.level + 1, ctx.N), dtype=np.uint64)
    lib().orc_relinearize(ctx._h, _p(_u64(d.data)), d.level, _p(keys.rlk), _p(out))
    return Ct(out, d.level, d.scale)


def rescale(ctx: Ctx, ct: Ct) -> Ct:
    if ct.level < 1:
        raise ValueError("rescale at level 0")
    npol = ct.data.shape[0]
    out = np.empty((npol, ct.level, ctx.N), dtype=np.uint64)
    lib().orc_rescale(ctx._h, _p(_u64(ct.data)), ct.level, npol, _p(out))
    return Ct(out, ct.level - 1, ct.scale / ctx.q[ct.level])


def mask(ctx: Ctx, ct: Ct, mask_key: bytes, ct_id: int):
    """Server half of Alg. 1: (masked [2][N] coef mod q0, share [N] = -r mod q0)."""
    masked = np.empty((2, ctx.N), dtype=np.uint64)
    share = np.empty(ctx.N, dtype=np.uint64)
    lib().orc_mask(ctx._h, _p(_u64(ct.data)), ct.level, mask_key, ct_id, _p(masked), _p(share))
    return masked, share


# ---------------------------------------------------------------------------
# S13: optional re-randomisation before the mask (reading C22)
# ---------------------------------------------------------------------------
def public_key(ctx: Ctx, key: bytes, s_ntt: np.ndarray) -> Ct:
    """The client's public key: a symmetric encryption of zero (C6) at the top level, id PK_ID:
    (b, a) = (-a s + e, a)."""
    zero = np.zeros((ctx.K, ctx.N), dtype=np.uint64)
    return encrypt(ctx, key, s_ntt, zero, ctx.K - 1, PK_ID, 1.0)


def flood_draws(key: bytes, objid: int, N: int, flood_bits: int) -> np.ndarray:
    """e0: uniform integers in [-2^f, 2^f) from the low bits of the 128-bit draws (f >= 1), or the
    centred binomial of C4 for f = 0 (plain re-randomisation)."""
    if flood_bits == 0:
        return sample_cbd(key, TAG_RR_E0, objid, N)
    m = (1 << (flood_bits + 1)) - 1
    return np.array([(draw128(key, TAG_RR_E0, objid, x) & m) - (1 << flood_bits) for x in range(N)], dtype=np.int64)


def rerandomize(ctx: Ctx, ct: Ct, pk: Ct, rr_key: bytes, ct_id: int, flood_bits: int) -> Ct:
    """S13 (paper silent, reading C22): drop to q_0, then add a fresh public-key encryption of zero
    with flooding noise, (v b + e0, v a + e1) mod q_0, v ternary, e1 centred binomial, e0 flooding
    (flood_draws); all draws keyed by the conversion's own id (ct_id << 8)."""
    oid = ct_id << 8
    c = Ct(ct.data[:, :1].copy(), 0, ct.scale)
    q0 = ctx.mods[0]

    def ntt0(v):
        return ctx.ntt(np.array([int(x) % q0 for x in v], dtype=np.uint64)[None, :], [0])[0]

    v = ntt0(sample_ternary(rr_key, TAG_RR_V, oid, ctx.N))
    e0 = ntt0(flood_draws(rr_key, oid, ctx.N, flood_bits))
    e1 = ntt0(sample_cbd(rr_key, TAG_RR_E1, oid, ctx.N))
    vpk = mul_pt(ctx, Ct(pk.data[:, :1].copy(), 0, 1.0), v[None, :], 1.0)
    z = add(ctx, vpk, Ct(np.stack([e0, e1])[:, None, :], 0, 1.0))
    return Ct(add(ctx, c, Ct(z.data, 0, c.scale)).data, 0, ct.scale)


# ---------------------------------------------------------------------------
# row f2: other HE operators of the fused blocks
# ---------------------------------------------------------------------------
def mul_relin(ctx: Ctx, a: Ct, b: Ct, keys: Keys) -> Ct:
    """ewmul_cc (Table 2): relinearised ct x ct product (C9), no rescale."""
    return relinearize(ctx, tensor(ctx, a, b), keys)


def rotate_sum(ctx: Ctx, ct: Ct, keys: Keys, L: int, D: int, broadcast: bool = False) -> Ct:
    """m^0 = m, m^i = m^{i-1} + Rot^{2^{i-1} L}(m^{i-1}), i = 1..log2 D (left
    rotations for sum, right rotations for broadcast); the fused form (no mask)."""
    assert D > 0 and D & (D - 1) == 0
    cur = ct.copy()
    step = L
    while step < L * D:
        cur = add(ctx, cur, rotate(ctx, cur, keys, -step if broadcast else step))
        step *= 2
    return cur


# ---------------------------------------------------------------------------
# extended basis Q_l u P (double hoisting, reading C13)
# ---------------------------------------------------------------------------
@dataclass
class CtExt:
    data: np.ndarray  # [2][level+1+np][N], NTT, over q_0..q_level, p_0..
    level: int
    scale: float


def ext_pidx(ctx: Ctx, level: int) -> list[int]:
    return list(range(level + 1)) + [ctx.K + t for t in range(ctx.np_)]


def rotate_ext(ctx: Ctx, ct: Ct, keys: Keys, step: int) -> CtExt:
    """Rotation kept in Q_l u P (no ModDown): (P sigma(c0) + u0, u1); step 0 lifts (P c0, P c1)."""
    g = ctx.galois(step)
    E = ct.level + 1 + ctx.np_
    out = np.empty((2, E, ctx.N), dtype=np.uint64)
    rk = keys.rot[g] if g != 1 else np.zeros(1, dtype=np.uint64)
    lib().orc_rotate_ext(ctx._h, _p(_u64(ct.data)), ct.level, _p(rk), g, _p(out))
    return CtExt(out, ct.level, ct.scale)


def encode_ext(ctx: Ctx, z, scale: float, level: int) -> np.ndarray:
    z = np.ascontiguousarray(z, dtype=np.float64)
    out = np.empty((level + 1 + ctx.np_, ctx.N), dtype=np.uint64)
    if lib().orc_encode_ext(ctx._h, _p(z), float(scale), level, _p(out)) != 0:
        raise EncodeOverflow("encode magnitude >= 2^62")
    return out


def mul_pt_ext(ctx: Ctx, a: CtExt, pt: np.ndarray, pt_scale: float) -> CtExt:
    idx = ext_pidx(ctx, a.level)
    pa = (ctypes.c_int * len(idx))(*idx)
    out = np.empty_like(a.data)
    lib().orc_mul_pt_idx(ctx._h, _p(_u64(a.data)), _p(_u64(pt)), pa, len(idx), 2, _p(out))
    return CtExt(out, a.level, a.scale * pt_scale)


def add_ext(ctx: Ctx, a: CtExt, b: CtExt) -> CtExt:
    idx = ext_pidx(ctx, a.level)
    pa = (ctypes.c_int * len(idx))(*idx)
    out = np.empty_like(a.data)
    lib().orc_add_idx(ctx._h, _p(_u64(a.data)), _p(_u64(b.data)), pa, len(idx), 2, _p(out))
    return CtExt(out, a.level, a.scale)


def relinearize_ext(ctx: Ctx, d: Ct, keys: Keys) -> CtExt:
    """Relinearisation kept in Q_l u P: (P d0 + u0, P d1 + u1) (reading C17)."""
    out = np.empty((2, d.level + 1 + ctx.np_, ctx.N), dtype=np.uint64)
    lib().orc_relinearize_ext(ctx._h, _p(_u64(d.data)), d.level, _p(keys.rlk), _p(out))
    return CtExt(out, d.level, d.scale)


def moddown_rescale(ctx: Ctx, a: CtExt) -> Ct:
    """ModDown fused with rescale (reading C17): round(X / (q_l P)) exactly, level l -> l - 1,
    scale / q_l (the P factor of the extended form is the lift's, not the message's)."""
    out = np.empty((2, a.level, ctx.N), dtype=np.uint64)
    lib().orc_moddown_rescale(ctx._h, _p(_u64(a.data)), a.level, _p(out))
    return Ct(out, a.level - 1, a.scale / ctx.q[a.level])


def moddown_ct(ctx: Ctx, a: CtExt) -> Ct:
    """ModDown of both polynomials (C7): back to Q_l, divided by P."""
    return Ct(np.stack([moddown(ctx, a.data[0], a.level), moddown(ctx, a.data[1], a.level)]), a.level, a.scale)


# ---------------------------------------------------------------------------
# f3: MPC -> CKKS ingest (Algorithm 2; ring-to-field, App. C.3)
# ---------------------------------------------------------------------------
def share_to_rns(ctx: Ctx, x, w: int, sub: bool, level: int) -> np.ndarray:
    """[x]^q = x mod q (P0) or x - 2^w mod q (P1, sub) per limb, NTT form [level+1][N].
    x: uint64 [N] (w <= 64) or [N][2] little-endian words (w <= 128, e.g. l + 40 = 83)."""
    x = np.ascontiguousarray(x, dtype=np.uint64)
    out = np.empty((level + 1, ctx.N), dtype=np.uint64)
    if x.ndim == 2:
        assert x.shape == (ctx.N, 2) and 1 <= w <= 128
        lib().orc_share_to_rns128(ctx._h, _p(x), int(w), int(bool(sub)), level, _p(out))
        return out
    assert x.shape == (ctx.N,) and 1 <= w <= 64
    lib().orc_share_to_rns(ctx._h, _p(x), int(w), int(bool(sub)), level, _p(out))
    return out


def mpc_to_ckks(ctx: Ctx, ct: Ct, x1, w: int) -> Ct:
    """Server half of Alg. 2 line 4: Enc([tmp]_0^q) (+) [tmp]_1^q, i.e. c0 += NTT(x1 - 2^w mod q_i)."""
    s = share_to_rns(ctx, x1, w, True, ct.level)
    idx = list(range(ct.level + 1))
    pa = (ctypes.c_int * len(idx))(*idx)
    c0 = np.empty_like(s)
    lib().orc_add_idx(ctx._h, _p(_u64(ct.data[0])), _p(s), pa, len(idx), 1, _p(c0))
    return Ct(np.stack([c0, ct.data[1].copy()]), ct.level, ct.scale)


def share_decode(ctx: Ctx, x: np.ndarray, ft: int, s_out: int) -> np.ndarray:
    """Row f3: local fixed-point Decode of a share over Z_{2^128} (x: uint64 [N][2] = lo, hi words)
    -> uint64 [N/2][2] share of the real slots scaled by 2^-s_out (reading C18)."""
    x = np.ascontiguousarray(x, dtype=np.uint64)
    assert x.shape == (ctx.N, 2) and 1 <= ft <= 62 and 0 <= s_out < 127
    y = np.empty((ctx.n, 2), dtype=np.uint64)
    lib().orc_share_decode(ctx._h, _p(x), int(ft), int(s_out), _p(y))
    return y


def share_encode(ctx: Ctx, y: np.ndarray, ft: int, s_out: int) -> np.ndarray:
    """Row f3 (Alg. 2 line 1): local fixed-point Encode of a slot-vector share over Z_{2^128}
    (y: uint64 [N/2][2]) -> uint64 [N][2] share of the integer coefficients (reading C20)."""
    y = np.ascontiguousarray(y, dtype=np.uint64)
    assert y.shape == (ctx.n, 2) and 1 <= ft <= 62 and 0 <= s_out < 127
    x = np.empty((ctx.N, 2), dtype=np.uint64)
    lib().orc_share_encode(ctx._h, _p(y), int(ft), int(s_out), _p(x))
    return x


def u128_to_int(a: np.ndarray) -> list[int]:
    """[..][2] uint64 words -> signed Python ints (two's complement, 128 bits)."""
    out = []
    for lo, hi in a.reshape(-1, 2):
        v = int(lo) | (int(hi) << 64)
        out.append(v - (1 << 128) if v >> 127 else v)
    return out


def int_to_u128(vals) -> np.ndarray:
    a = np.empty((len(vals), 2), dtype=np.uint64)
    for i, v in enumerate(vals):
        v %= 1 << 128
        a[i, 0], a[i, 1] = v & (2 ** 64 - 1), v >> 64
    return a
