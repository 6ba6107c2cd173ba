"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no encoding, no modular
arithmetic, no packing): only numpy PCG64 draws of float matrices with the
shapes and distributions of the paper's workloads, the 32-byte ChaCha20 keys
derived from integer seeds, and the preset parameter *widths* (each side derives
its own primes from them).  Recipe: DESIGN.md "Input recipe".
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np


def crypto_key(seed: int, config_id: int) -> bytes:
    """key = LE64(seed) || LE64(config id) || 16 zero bytes."""
    return struct.pack("<QQ", seed & (2**64 - 1), config_id & (2**64 - 1)) + bytes(16)


@dataclass(frozen=True)
class Preset:
    name: str
    log_n: int
    q_bits: tuple
    p_bits: tuple
    dnum: int
    log_delta: int

    @property
    def N(self):
        return 1 << self.log_n

    @property
    def n(self):
        return 1 << (self.log_n - 1)


# config 1 (toy, insecure): Q = {60, 40, 40}, P = {60}, dnum = 3, Delta = 2^40
TOY = Preset("toy", 12, (60, 40, 40), (60,), 3, 40)
# configs 2-5: N = 2^16, Q = {60, 40 x 4}, P = {60}, dnum = 5 (alpha = 1), Delta = 2^40
BERT = Preset("bert", 16, (60, 40, 40, 40, 40), (60,), 5, 40)
# the config-2 dnum = 1 variant (reading C23): one key-switch digit = all of Q (220 bits),
# so P must exceed it: four 60-bit special primes (240 bits; log QP = 460, inside the N = 2^16 bound)
BERT_DNUM1 = Preset("bert_dnum1", 16, (60, 40, 40, 40, 40), (60, 60, 60, 60), 1, 40)
# small presets used only by tests (a ragged/tiny ring, and alpha = 2 digits)
TINY = Preset("tiny", 5, (50, 40, 40), (60,), 3, 30)
MID = Preset("mid", 10, (60, 40, 40, 40), (61, 61), 2, 36)


def rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


def uniform(seed: int, shape, lo: float, hi: float) -> np.ndarray:
    return rng(seed).uniform(lo, hi, size=shape).astype(np.float64)


def normal(seed: int, shape, std: float, clip: float | None = None) -> np.ndarray:
    x = rng(seed).normal(0.0, std, size=shape)
    if clip is not None:
        x = np.clip(x, -clip, clip)
    return x.astype(np.float64)


def gelu(x: np.ndarray) -> np.ndarray:
    from math import erf, sqrt
    v = np.vectorize(lambda t: 0.5 * t * (1.0 + erf(t / sqrt(2.0))))
    return v(x).astype(np.float64)


# ---- config 1: toy ct-pt 16x16x16 + mask ---------------------------------
def toy_inputs():
    X = uniform(1, (16, 16), -1.0, 1.0)
    W = uniform(2, (16, 16), -0.5, 0.5)
    return dict(X=X, W=W, mask_key=crypto_key(3, 1), keys_key=crypto_key(4, 1), enc_key=crypto_key(5, 1))


# ---- config 2: BERT-base attention (QKV + Q K^T) --------------------------
BERT_BASE = dict(L=128, d=768, H=12, ffn=3072)
BERT_LARGE = dict(L=128, d=1024, H=16, ffn=4096)
GPT2_BASE = dict(L=128, d=768, H=12, ffn=3072)
# BSGS baby-step counts B of the layer plans bench.py times (C11 plan parameter, reading S15;
# 0 = the ct-ct default B = g).  A workload parameter, not arithmetic: bench.py and the
# full-size parity tests (tests/test_gpu_bert.py) both read it, so they cannot drift apart.
# (QKV at B = 32: 7.6-7.7 vs 7.8-8.0 ms per layer at B = 64, profiles/r2s2_bsgs_sweep.log; FFN1 equal)
BENCH_BSGS = {"qkv": 32, "oproj": 16, "ffn1": 64, "ffn2": 16, "qk": 0}


def bert_attention_inputs(L=128, d=768, config_id=2):
    X = normal(11, (L, d), 1.0, clip=4.0)
    WQ = normal(12, (d, d), 0.04)
    WK = normal(13, (d, d), 0.04)
    WV = normal(14, (d, d), 0.04)
    return dict(X=X, WQ=WQ, WK=WK, WV=WV, keys_key=crypto_key(4, config_id),
                enc_key=crypto_key(5, config_id), mask_key=crypto_key(3, config_id))


# ---- config 3: out-proj (diagonal input) + FFN ----------------------------
def softmax_rows(x: np.ndarray) -> np.ndarray:
    e = np.exp(x - x.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def bert_ffn_inputs(L=128, d=768, H=12, ffn=3072, config_id=3):
    dh = d // H
    Att = normal(21, (H, L, dh), 1.0)
    S = softmax_rows(normal(28, (H, L, L), 1.0))      # Softmax(Q K^T / sqrt(d_h)) rows (f1 operand)
    V = normal(27, (H, L, dh), 1.0)
    WO = normal(22, (d, d), 0.04)
    X2 = normal(23, (L, d), 1.0)
    W1 = normal(24, (d, ffn), 0.04)
    H1 = gelu(normal(25, (L, ffn), 1.0))
    W2 = normal(26, (ffn, d), 0.02)
    return dict(Att=Att, S=S, V=V, WO=WO, X2=X2, W1=W1, H1=H1, W2=W2, keys_key=crypto_key(4, config_id),
                enc_key=crypto_key(5, config_id), mask_key=crypto_key(3, config_id))


# a toy ring with the BERT chain shape (5 ciphertext primes): room for QKV + Q K^T (depth 4)
QKTOY = Preset("qktoy", 12, (60, 40, 40, 40, 40), (60,), 5, 40)
QKTOY_DNUM1 = Preset("qktoy_dnum1", 12, (60, 40, 40, 40, 40), (60, 60, 60, 60), 1, 40)


def qk_toy_inputs(H=4, L=32, dh=32):
    Q = uniform(41, (H, L, dh), -1.0, 1.0)
    K = uniform(42, (H, L, dh), -1.0, 1.0)
    return dict(Q=Q, K=K, keys_key=crypto_key(4, 41), enc_key=crypto_key(5, 41), mask_key=crypto_key(3, 41))


# ---- row f2: fused-block chains ---------------------------------------------
# BOLT's GeLU approximation a|x|^4 + b|x|^3 + c|x|^2 + d|x| + e + 0.5 x on |x| <= 2.7;
# the paper defers the coefficients to BOLT, so they are fitted here (reading C21): least squares of
# 0.5 x erf(x / sqrt 2) on 20001 points of [0, 2.7] (max error 4.2e-3).  A workload parameter.
GELU_COEF = (0.023453955861263417, -0.19812474039214562, 0.5675004464374074, -0.05485410511200729,
             0.004240801424024679)
# Table 6 block 3 preset: N = 32768, RNS {60, 40 x 7, 60}, scale 40 (depth 7); the f2
# chains run on it (reading C21)
F2 = Preset("f2", 15, (60, 40, 40, 40, 40, 40, 40, 40), (60,), 8, 40)
# the same chain shape on a small ring for parity tests
F2TOY = Preset("f2toy", 12, (60, 40, 40, 40, 40, 40, 40, 40), (60,), 8, 40)
