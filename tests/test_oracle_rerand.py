"""S13 (reading C22) oracle pins: the public key is an encryption of zero; the re-randomised
level-0 ciphertext differs from the input in decryption by exactly v e_pk + e0 + e1 s (schoolbook
negacyclic products), with v ternary, e1 centred binomial and |e0| <= 2^f; the CKKS->MPC
shares still reconstruct the (re-randomised) decryption exactly (Alg. 1)."""
import numpy as np
import pytest

import blb_inputs as bi
import oracle as O


@pytest.fixture(scope="module")
def toy():
    P = bi.TOY
    pr = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    ctx = O.Ctx(P.log_n, pr[:3], pr[3:], P.dnum)
    keys = O.keygen(ctx, bi.crypto_key(4, 60))
    return ctx, keys


def centred(v, q):
    v = [int(x) for x in v]
    return [x - q if x > q // 2 else x for x in v]


@pytest.mark.parametrize("flood", [0, 20])
def test_rerandomisation_adds_exactly_a_fresh_zero(toy, flood):
    ctx, keys = toy
    q0 = ctx.mods[0]
    pk = O.public_key(ctx, bi.crypto_key(5, 60), keys.s_ntt)
    e_pk = centred(ctx.intt(O.decrypt(ctx, keys.s_ntt, pk)[:1], [0])[0], q0)
    assert max(abs(x) for x in e_pk) <= 21                      # C4: CBD eta = 21
    z = np.random.default_rng(61).uniform(-1, 1, ctx.n)
    ct = O.encrypt(ctx, bi.crypto_key(5, 60), keys.s_ntt, O.encode(ctx, z, 2.0 ** 40, 2), 2, 7, 2.0 ** 40)
    rr_key, cid = bi.crypto_key(6, 60), 1234
    rr = O.rerandomize(ctx, ct, pk, rr_key, cid, flood)
    d_rr = ctx.intt(O.decrypt(ctx, keys.s_ntt, rr), [0])[0]
    d_ct = ctx.intt(O.decrypt(ctx, keys.s_ntt, O.Ct(ct.data[:, :1].copy(), 0, ct.scale)), [0])[0]
    v = O.sample_ternary(rr_key, O.TAG_RR_V, cid << 8, ctx.N)
    e1 = O.sample_cbd(rr_key, O.TAG_RR_E1, cid << 8, ctx.N)
    e0 = O.flood_draws(rr_key, cid << 8, ctx.N, flood)
    assert set(np.unique(v)) <= {-1, 0, 1}
    assert np.abs(e0).max() <= (2 ** flood if flood else 21)
    s = [int(x) for x in keys.s_coef]
    to_q = lambda a: np.array([int(x) % q0 for x in a], dtype=np.uint64)  # noqa: E731
    ve = O.schoolbook(to_q(v), to_q(e_pk), q0)
    e1s = O.schoolbook(to_q(e1), to_q(s), q0)
    want = [(int(a) + int(b) + int(c)) % q0 for a, b, c in zip(ve, e1s, to_q(e0))]
    got = [(int(a) - int(b)) % q0 for a, b in zip(d_rr, d_ct)]
    assert got == want
    # the shares of the re-randomised ciphertext reconstruct its decryption exactly (C14)
    masked, share = O.mask(ctx, rr, bi.crypto_key(3, 60), cid)
    s0 = keys.s_ntt[0]
    tmp0 = ctx.intt(((ctx.ntt(masked[0][None, :], [0])[0].astype(object) +
                      ctx.ntt(masked[1][None, :], [0])[0].astype(object) * s0.astype(object)) % q0)
                    .astype(np.uint64)[None, :], [0])[0]
    rec = [(int(a) + int(b)) % q0 for a, b in zip(tmp0, share)]
    assert rec == [int(x) for x in d_rr]
    # flooding keeps the message: decode error of 2^f noise at Delta = 2^40
    dec = O.decode(ctx, O.decrypt(ctx, keys.s_ntt, rr), rr.scale)
    assert np.abs(dec - z).max() < 2.0 ** -10
