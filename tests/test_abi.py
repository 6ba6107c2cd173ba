"""C-ABI boundary checks that need no GPU: libblb.so loads, exports every symbol
include/blb.h declares, and its host-only helpers agree with the paper-derived
KATs (C1 prime rule) and with the oracle's independent MHP map."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def blb():
    import paper_2508_19525_b200 as blb
    blb.build()
    return blb


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "blb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(blb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(blb):
    L = ctypes.CDLL(blb.SO)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_library_is_sm100a(blb):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", blb.SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_prime_chain_host_helper(blb):
    kat = json.load(open(os.path.join(ROOT, "tests", "golden", "kat_primes.json")))
    for name in ("toy", "bert"):
        assert blb.prime_chain(kat[name]["log_n"], kat[name]["bits"]) == kat[name]["primes"]
    with pytest.raises(blb.BLBError):
        blb.prime_chain(12, [62])


def test_mhp_map_matches_oracle(blb):
    import oracle.matmul as mm
    for d, H, L, logn in [(768, 12, 128, 16), (1024, 16, 128, 16), (8, 2, 4, 5), (64, 4, 16, 12)]:
        assert blb.mhp_column_map(d, H, L, logn) == mm.mhp_column_map(d, H, L, 1 << (logn - 1))


def test_packing_matches_oracle_layout(blb):
    from paper_2508_19525_b200 import packing
    import oracle.matmul as mm
    X = np.random.default_rng(0).normal(size=(16, 300))
    assert np.array_equal(packing.spatial_slots(X, 2048), np.stack(mm.pack_spatial(X, 2048)))
    assert np.array_equal(packing.spatial_unslots(packing.spatial_slots(X, 2048), 16, 300), X)
    A = np.random.default_rng(1).normal(size=(4, 16, 8))
    assert np.array_equal(packing.diagonal_slots(A, 512), np.stack(mm.pack_diagonal_mh(A, 512)))


def test_mhp_packing_matches_oracle_layout(blb):
    from paper_2508_19525_b200 import packing
    import oracle.matmul_cc as cc
    rng = np.random.default_rng(3)
    for H, L, D, n in [(3, 32, 16, 2048), (12, 128, 64, 32768), (4, 16, 16, 512)]:
        M = rng.normal(size=(H, L, D))
        assert np.array_equal(packing.mhp_slots(M, n), np.stack(cc.pack_mhp(M, cc.plan_qk(L, H, D, n))))
        S, V = rng.normal(size=(H, L, L)), rng.normal(size=(H, L, L // 2))
        a, k = packing.softmax_v_operands(S, V, n)
        A, K = cc.sv_operands(S, V)
        p = cc.plan_sv(L, H, n)
        assert np.array_equal(a, np.stack(cc.pack_mhp(A, p))) and np.array_equal(k, np.stack(cc.pack_mhp(K, p)))
