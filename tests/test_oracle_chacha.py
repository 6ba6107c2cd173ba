"""Oracle pins: ChaCha20 (RFC 8439 sec. 2.3) and the C4 draw layout, checked
against the independent `cryptography` implementation; mask KAT (C14)."""
import json
import os
import struct

import numpy as np
import pytest
from cryptography.hazmat.primitives.ciphers import Cipher, algorithms

import oracle as O

MASK_KAT = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "mask_kat.json")))


def keystream(key: bytes, counter: int, nonce12: bytes, nbytes: int) -> bytes:
    enc = Cipher(algorithms.ChaCha20(key, struct.pack("<I", counter) + nonce12), mode=None).encryptor()
    return enc.update(bytes(nbytes))


def ref_draw(key, tag, objid, x):
    nonce = struct.pack("<IQ", tag, objid)
    blk = keystream(key, x // 4, nonce, 64)
    d = x % 4
    return int.from_bytes(blk[16 * d:16 * d + 16], "little")


def test_rfc8439_block_vector():
    key = bytes(range(32))
    nonce = bytes.fromhex("000000090000004a00000000")
    out = O.chacha20_block(key, 1, nonce)
    assert out == keystream(key, 1, nonce, 64)
    assert out[:16].hex() == "10f1e7e4d13b5915500fdd1fa32071c4"  # RFC 8439 sec. 2.3.2


def test_block_random_vs_cryptography():
    rng = np.random.default_rng(0)
    for _ in range(20):
        key = rng.bytes(32)
        nonce = rng.bytes(12)
        ctr = int(rng.integers(0, 2**32))
        assert O.chacha20_block(key, ctr, nonce) == keystream(key, ctr, nonce, 64)


def test_draw_layout():
    key = bytes(range(32))
    for tag, objid in [(6, 0), (2, (5 << 8) | 3), (4, 2**40 + 7)]:
        for x in [0, 1, 2, 3, 4, 5, 1023]:
            assert O.draw128(key, tag, objid, x) == ref_draw(key, tag, objid, x)


def test_samplers_match_definition():
    key = bytes(range(1, 33))
    N, q = 64, 1099511480321
    u = O.sample_uniform(key, 2, 77, q, N)
    t = O.sample_ternary(key, 1, 0, N)
    e = O.sample_cbd(key, 3, 9 << 8, N)
    m21 = (1 << 21) - 1
    for x in range(N):
        assert int(u[x]) == ref_draw(key, 2, 77, x) % q
        lo = ref_draw(key, 1, 0, x) & (2**64 - 1)
        assert int(t[x]) == lo % 3 - 1
        lo = ref_draw(key, 3, 9 << 8, x) & (2**64 - 1)
        assert int(e[x]) == bin(lo & m21).count("1") - bin((lo >> 21) & m21).count("1")
    assert set(t.tolist()) <= {-1, 0, 1}
    assert np.abs(e).max() <= 21


@pytest.mark.parametrize("row", MASK_KAT["rows"], ids=lambda r: "%s-%d" % (r["preset"], r["ct_id"]))
def test_mask_kat(row):
    key = bytes(range(32))
    q0 = row["q0"]
    objid = row["ct_id"] << 8
    got = O.sample_uniform(key, O.TAG_MASK, objid, q0, 4)
    assert [int(v) for v in got] == row["r"]
    assert [ref_draw(key, 6, objid, x) % q0 for x in range(4)] == row["r"]
