"""Oracle ct-ct MatMul Q_h K_h^T for all heads -- TEST INFRASTRUCTURE ONLY.

BLB's rotation-efficient ct-ct protocol (sec. 5.1): Observations 1-2
(P:448-451), the three steps, multi-head packing (MHP)
and BSGS with the giant step deferred into step 3 (App. C.1).  The
paper does not pin every mask (fig:matmul_cc and fig:bsgs are elided), so this
is the reconstruction of DESIGN.md reading C13, written at the slot level with
numpy and executed with the oracle's CKKS primitives:

MHP layout (L, H_p, g): block beta = c*H_p + h (c < g) of ciphertext j holds
column k = j*g + c of head h (rows p = 0..L-1 contiguous); g = n / (L H_p),
J = d_h / g ciphertexts each for Q and K (both spatial-first, so K is K^T in
reduce-first packing).  With t = u*B + i (u < G, i < B, B*G = L, g | B):

  baby (steps 1+2, K side): K'_i = inner rotation of block (c, h) by c + i:
       ModDown( sum_c Mnw_{c,i} (.) Rot_s(K) + Mw_{c,i} (.) Rot_{s-L}(K) ), s = (c+i) mod L,
       the rotations double-hoisted (one ModUp, kept in Q_l u P, one ModDown per K'_i)
  giant (Q side):           Q_u  = inner rotation by -uB:
       ModDown( Mq1_u (.) Rot_{-uB}(Q) + Mq2_u (.) Rot_{L-uB}(Q) ) (same double hoisting)
  products:                 S_{u,i} = relin( sum_j Q_u^(j) (x) K'_i^(j) )
       -> block (c,h), row p: partial_{k == c mod g} C_h[p - uB, p + uB + i + c - uB]
  step 3:                   T_{u,i} = Rot_{-i H_p L}(S_{u,i})   (right by i block-groups)
       A_{u,w,f} = sum_i M3_{u,i,w,f} (.) T_{u,i}: block c' has wrap class
       w = (c + i) div g (c = (c'-i) mod g) and source rows p >= uB (f=0) / < uB (f=1)
  deferred giant fix:       Rot_{uB}(A_{u,w,0}),  Rot_{uB-L}(A_{u,w,1})
  output o = ((uB + w g) mod L) / g: block e*H_p + h, row p of output o holds
       C_h[p, (p + o g + e) mod L]   (diagonal packing)

Masks are encoded at the scale of the prime the next rescale drops; every mask
stage is followed by one rescale; the product stage by relinearisation and one
rescale: depth 3 here + 1 for the QKV ct-pt MatMul = 4.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

import oracle as O

from . import Ct, Ctx, Keys, add, encode, mul_pt, relinearize, rescale, rotate, tensor


@dataclass
class QKPlan:
    L: int
    H: int
    Hp: int
    dh: int
    n: int
    g: int
    J: int
    B: int
    G: int
    # rotation amounts (slots, left positive)
    k_rots: list = field(default_factory=list)
    q_rots: list = field(default_factory=list)

    @property
    def n_out(self) -> int:
        return self.L // self.g

    def block_c(self) -> np.ndarray:
        """c index of every slot."""
        s = np.arange(self.n)
        return (s // self.L) // self.Hp

    def pos(self) -> np.ndarray:
        return np.arange(self.n) % self.L

    # ---- masks (0/1 slot vectors) ----
    def mask_k(self, c: int, i: int, wrap: bool) -> np.ndarray:
        s = (c + i) % self.L
        cc, p = self.block_c(), self.pos()
        sel = (cc == c) & ((p + s >= self.L) if wrap else (p + s < self.L))
        return sel.astype(np.float64)

    def mask_q(self, u: int, low: bool) -> np.ndarray:
        a = u * self.B
        p = self.pos()
        return ((p < a) if low else (p >= a)).astype(np.float64)

    def wrap_class(self, cprime: int, i: int) -> int:
        c = (cprime - i) % self.g
        return (c + i) // self.g

    def mask3(self, u: int, i: int, w: int, f: int) -> np.ndarray:
        cc, p = self.block_c(), self.pos()
        wc = np.array([self.wrap_class(x, i) for x in range(self.g)])[cc]
        a = u * self.B
        sel = (wc == w) & ((p >= a) if f == 0 else (p < a))
        return sel.astype(np.float64)

    def accumulators(self):
        """(u, w, f) triples with at least one non-zero step-3 mask."""
        out = []
        wmax = (self.g - 1 + self.B - 1) // self.g
        for u in range(self.G):
            for w in range(wmax + 1):
                for f in (0, 1):
                    if any(self.mask3(u, i, w, f).any() for i in range(self.B)):
                        out.append((u, w, f))
        return out

    def out_index(self, u: int, w: int) -> int:
        return ((u * self.B + w * self.g) % self.L) // self.g

    def final_rot(self, u: int, f: int) -> int:
        return u * self.B if f == 0 else u * self.B - self.L

    def rotation_steps(self) -> list[int]:
        s = set(self.k_rots) | set(self.q_rots)
        # step-3 rotations by a multiple of n slots are the identity sigma_1 (no key, C13)
        s |= {-i * self.Hp * self.L for i in range(1, self.B) if (i * self.Hp * self.L) % self.n}
        for u, w, f in self.accumulators():
            r = self.final_rot(u, f)
            if r % self.n:
                s.add(r)
        s.discard(0)
        return sorted(s)

    def counts(self) -> dict:
        n_k = self.J * len([r for r in self.k_rots if r % self.n])
        n_q = self.J * len([r for r in self.q_rots if r % self.n])
        n_3 = self.G * len([i for i in range(1, self.B) if (i * self.Hp * self.L) % self.n])
        n_f = len([1 for u, w, f in self.accumulators() if self.final_rot(u, f) % self.n])
        return {"rotations": n_k + n_q + n_3 + n_f, "baby": n_k, "giant": n_q, "step3": n_3, "final": n_f,
                "cmult": self.G * self.B * self.J, "relin": self.G * self.B}


def plan_qk(L: int, H: int, dh: int, n: int, B: int | None = None) -> QKPlan:
    Hp = 1 << (H - 1).bit_length()
    g = n // (L * Hp)
    assert g >= 1 and g * L * Hp == n, "MHP needs n = g * L * H_p"
    J = math.ceil(dh / g)
    B = g if B is None else B
    assert B % g == 0 and L % B == 0, "reading C13 needs g | B | L"
    G = L // B
    plan = QKPlan(L, H, Hp, dh, n, g, J, B, G)
    ks = set()
    for c in range(g):
        for i in range(B):
            s = (c + i) % L
            if s:
                ks.add(s)
                ks.add(s - L)
    plan.k_rots = sorted(ks)
    qs = set()
    for u in range(1, G):
        qs.add(-u * B)
        qs.add(L - u * B)
    plan.q_rots = sorted(qs)
    return plan


def pack_mhp(M: np.ndarray, plan: QKPlan) -> list[np.ndarray]:
    """M: (H, L, d_h) -> J slot vectors; block c*H_p + h of ciphertext j = column j*g + c of head h."""
    H, L, dh = M.shape
    out = []
    for j in range(plan.J):
        z = np.zeros(plan.n)
        for c in range(plan.g):
            k = j * plan.g + c
            if k >= dh:
                continue
            for h in range(H):
                b = c * plan.Hp + h
                z[b * L:(b + 1) * L] = M[h, :, k]
        out.append(z)
    return out


def unpack_diag(outs: list[np.ndarray], plan: QKPlan) -> np.ndarray:
    """Output slot vectors -> C (H, L, L) with C_h[p, (p + d) mod L] from diagonal d."""
    L = plan.L
    C = np.zeros((plan.H, L, L))
    p = np.arange(L)
    for o, z in enumerate(outs):
        for e in range(plan.g):
            d = o * plan.g + e
            for h in range(plan.H):
                b = e * plan.Hp + h
                C[h, p, (p + d) % L] = z[b * L:(b + 1) * L]
    return C


# ---------------------------------------------------------------------------
def slot_level(Qz: list[np.ndarray], Kz: list[np.ndarray], plan: QKPlan) -> list[np.ndarray]:
    """The same schedule on plaintext slot vectors (exactness pin)."""
    rot = lambda z, r: np.roll(z, -r)  # noqa: E731  left rotation by r
    Kp = {}
    for i in range(plan.B):
        for j in range(plan.J):
            acc = np.zeros(plan.n)
            for c in range(plan.g):
                s = (c + i) % plan.L
                acc += plan.mask_k(c, i, False) * rot(Kz[j], s)
                if s:
                    acc += plan.mask_k(c, i, True) * rot(Kz[j], s - plan.L)
            Kp[(i, j)] = acc
    Qu = {}
    for u in range(plan.G):
        for j in range(plan.J):
            if u == 0:
                Qu[(u, j)] = Qz[j].copy()
            else:
                a = u * plan.B
                Qu[(u, j)] = plan.mask_q(u, False) * rot(Qz[j], -a) + plan.mask_q(u, True) * rot(Qz[j], plan.L - a)
    outs = [np.zeros(plan.n) for _ in range(plan.n_out)]
    for u, w, f in plan.accumulators():
        A = np.zeros(plan.n)
        for i in range(plan.B):
            S = sum(Qu[(u, j)] * Kp[(i, j)] for j in range(plan.J))
            T = rot(S, -i * plan.Hp * plan.L)
            A += plan.mask3(u, i, w, f) * T
        outs[plan.out_index(u, w)] += rot(A, plan.final_rot(u, f))
    return outs


def qk_encrypted(ctx: Ctx, keys: Keys, Q: list[Ct], K: list[Ct], plan: QKPlan, out_ids=None) -> list[Ct]:
    """Evaluate the schedule on ciphertexts (all inputs at one level l >= 3).

    out_ids (optional): compute only these output ciphertexts (sampled parity at full size).  The
    schedule of each computed output is unchanged; only the giant steps u and step-3 accumulators
    that feed no requested output are skipped (every K'_i is still needed by every output)."""
    lvl = Q[0].level
    assert lvl >= 3 and all(c.level == lvl for c in Q + K)
    accs = plan.accumulators()
    if out_ids is not None:
        accs = [a for a in accs if plan.out_index(a[0], a[1]) in set(out_ids)]
    need_u = sorted({u for u, w, f in accs})

    def drop(ct: Ct) -> Ct:   # exact level drop (C9): keep limbs 0..level-1
        return Ct(ct.data[:, : ct.level].copy(), ct.level - 1, ct.scale)

    # Stage 1 is double-hoisted (reading C13): every rotation of K^(j) / Q^(j) shares one
    # ModUp and stays in the extended basis Q_l u P (no ModDown); the masks (encoded over
    # Q_l u P at scale q_l) are applied there and each masked sum gets ONE ModDown, then
    # one rescale -> level l-1.
    s1 = float(ctx.q[lvl])
    enc1 = {}

    def pt1(key, vec):
        if key not in enc1:
            enc1[key] = O.encode_ext(ctx, vec, s1, lvl)
        return enc1[key]

    Kp = {}
    for j in range(plan.J):
        rots = {r: O.rotate_ext(ctx, K[j], keys, r) for r in [0] + list(plan.k_rots)}
        for i in range(plan.B):
            acc = None
            for c in range(plan.g):
                s = (c + i) % plan.L
                parts = [(False, s)] + ([(True, s - plan.L)] if s else [])
                for wrap, r in parts:
                    term = O.mul_pt_ext(ctx, rots[r], pt1(("k", c, i, wrap), plan.mask_k(c, i, wrap)), s1)
                    acc = term if acc is None else O.add_ext(ctx, acc, term)
            Kp[(i, j)] = O.moddown_rescale(ctx, acc)
    Qu = {}
    for j in range(plan.J):
        Qu[(0, j)] = drop(Q[j])
        for u in need_u:
            if u == 0:
                continue
            a = u * plan.B
            t1 = O.mul_pt_ext(ctx, O.rotate_ext(ctx, Q[j], keys, -a), pt1(("q", u, False), plan.mask_q(u, False)), s1)
            t2 = O.mul_pt_ext(ctx, O.rotate_ext(ctx, Q[j], keys, plan.L - a),
                              pt1(("q", u, True), plan.mask_q(u, True)), s1)
            Qu[(u, j)] = O.moddown_rescale(ctx, O.add_ext(ctx, t1, t2))
    # products, relinearisation (once per (u, i), lazy over j: reading S10), rescale -> lvl-2
    T = {}
    for u in need_u:
        for i in range(plan.B):
            d = None
            for j in range(plan.J):
                t = tensor(ctx, Qu[(u, j)], Kp[(i, j)])
                d = t if d is None else add(ctx, d, t)
            S = O.moddown_rescale(ctx, O.relinearize_ext(ctx, d, keys))   # C17
            # step-3 rotation kept in Q u P (double hoisting, C13); i = 0 is the lift
            T[(u, i)] = O.rotate_ext(ctx, S, keys, -i * plan.Hp * plan.L)
    # step 3 masks at level lvl-2 (scale q_{lvl-2}) in Q u P, ModDown + rescale -> lvl-3 (C17),
    # final rotations summed in Q u P, one ModDown per output
    l3 = lvl - 2
    s3 = float(ctx.q[l3])
    outs = [None] * plan.n_out
    for u, w, f in accs:
        A = None
        for i in range(plan.B):
            m = plan.mask3(u, i, w, f)
            if not m.any():
                continue
            term = O.mul_pt_ext(ctx, T[(u, i)], O.encode_ext(ctx, m, s3, l3), s3)
            A = term if A is None else O.add_ext(ctx, A, term)
        A = O.moddown_rescale(ctx, A)
        Ae = O.rotate_ext(ctx, A, keys, plan.final_rot(u, f) % plan.n)
        o = plan.out_index(u, w)
        outs[o] = Ae if outs[o] is None else O.add_ext(ctx, outs[o], Ae)
    if out_ids is not None:
        return [O.moddown_ct(ctx, outs[o]) for o in out_ids]
    return [O.moddown_ct(ctx, e) for e in outs]


# ---------------------------------------------------------------------------
# f1: Softmax x V_h with zero padding d_h -> L, dense-diagonal collapse of
# adjacent outputs (fig:diag (b)), feeding the diagonal ct-pt W_O (C12)
# ---------------------------------------------------------------------------
def plan_sv(L: int, H: int, n: int, B: int | None = None) -> QKPlan:
    """C13 with inner dimension L: operands S_h (L x L) and Vpad_h^T (L x L)."""
    return plan_qk(L, H, L, n, B)


def sv_operands(S: np.ndarray, V: np.ndarray):
    """S: (H, L, L) softmax rows; V: (H, L, d_h) -> (A, Kop) both (H, L, L): C13 computes
    C[i, i+t] = sum_k A[i,k] Kop[i+t, k], so Kop = Vpad^T gives C = S Vpad."""
    H, L, dh = V.shape
    Vpad = np.zeros((H, L, L))
    Vpad[:, :, :dh] = V
    return S, np.transpose(Vpad, (0, 2, 1)).copy()


def collapse_dense(outs: list, plan: QKPlan, dh: int, add_fn=None) -> list:
    """Outputs o and o + n_out/2 hold diagonals d and d + d_h (d_h = L/2) with
    complementary support: their sum is the dense diagonal d of the L x d_h result."""
    assert 2 * dh == plan.L, "the collapse needs padding by exactly 2x (P:1213)"
    half = plan.n_out // 2
    add_fn = add_fn or (lambda a, b: a + b)
    return [add_fn(outs[o], outs[o + half]) for o in range(half)]


def pad_heads_rows(WO: np.ndarray, H: int, Hp: int) -> np.ndarray:
    """W_O rows reordered for the MHP-padded diagonal input: head h < H keeps its
    d_h rows, padded heads get zero rows."""
    D, Dout = WO.shape
    dh = D // H
    out = np.zeros((Hp * dh, Dout))
    out[:H * dh] = WO
    return out
