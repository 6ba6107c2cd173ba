"""Layer driver: the fused-linear CKKS evaluation of one Transformer layer
(BASELINE.json configs 2 + 3) on one rank of a data-parallel group.

Blocks (fig:fusion_pattern P:699-704, Table 6):
  * attention: QKV projection (C11, MHP reorder of the Q / K columns, P:466,
    P:511) -> Q K^T for all heads (row a7, reading C13) -> CKKS->MPC masks of
    the Q K^T diagonals and of V;
  * Softmax x V (row f1): the ct-ct protocol on the client-re-encrypted S_h and
    zero-padded V_h^T -> dense-diagonal collapse of adjacent outputs
     -> out-projection as the diagonal-input ct-pt MatMul (C12, App. C.2)
    with the MHP row reorder of W_O -> mask;
  * FFN1 (d -> 4d) -> mask; FFN2 (4d -> d) -> mask.
Each MatMul starts from a fresh ciphertext at the top level (SURVEY 8(d)
config 3).

Multi-GPU: every MatMul -- ct-pt and ct-ct -- is
sharded by its BSGS baby-step index i: rank r owns the contiguous window
shard(B, r, world) of [0, B), holds only the plaintexts of its window, computes the
baby-step rotations, MAC entries, products and step-3 terms of its window, and
writes its partial accumulators (ct-pt: acc_{b',g}; ct-ct: the step-3 A_{u,w,f} in
Q u P).  One exact all-reduce (u64 sums of residues < 2^61: no overflow for <= 8
ranks) adds the windows; the owner of each output ciphertext (shard(n_out, r,
world)) reduces mod q and runs the giant steps / ModDown / rescale and the mask.
Ciphertexts a later MatMul consumes whole (Q, K for Q K^T; the Softmax x V outputs
for the out-projection) are all-gathered.  The BSGS split does not depend on the
number of ranks and the sums are exact, so outputs are bit-identical at every GPU
count (tests/test_gpu_multirank.py).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

import paper_2508_19525_b200 as blb


def bi_log_delta() -> int:
    return 40


@dataclass
class Dims:
    L: int = 128
    d: int = 768
    H: int = 12
    ffn: int = 3072


BERT_BASE = Dims()
BERT_LARGE = Dims(128, 1024, 16, 4096)
BSGS = {"qkv": 32, "oproj": 16, "ffn1": 64, "ffn2": 16, "qk": 0}
# mask object ids (reading C19): id = seq * 2^24 + block * 2^16 + output, so every
# conversion of every inference draws a fresh mask (Alg. 1 line 1; Theorem 1)
MASK_BLOCK = {"qkv": 0, "oproj": 1, "ffn1": 2, "ffn2": 3, "qk": 4}
MAX_OUT = 1 << 16
MAX_SEQ = 1 << 32


def mask_id(seq: int, block: str, o: int) -> int:
    if not (0 <= o < MAX_OUT and 0 <= seq < MAX_SEQ):
        raise ValueError("mask id out of range: seq %d, output %d" % (seq, o))
    return (seq << 24) | (MASK_BLOCK[block] << 16) | o


def shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous split of n outputs over world ranks: (first, count)."""
    base, rem = divmod(n, world)
    first = rank * base + min(rank, rem)
    return first, base + (1 if rank < rem else 0)


def allgather_ragged(local: list, counts: list, like=None) -> list:
    """All-gather a rank-ordered ragged list (rank r holds counts[r] items, every item a
    tensor of one common shape) into the full list, ordered by rank, on every rank.
    One padded all_gather_into_tensor (NCCL over NVLink on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist
    world = len(counts)
    if world == 1:
        return list(local)
    ref = local[0] if local else like
    shape, dtype, device = ref.shape, ref.dtype, ref.device
    per = ref.numel()
    mx = max(counts)
    buf = torch.zeros(mx * per, dtype=dtype, device=device)
    for t, x in enumerate(local):
        buf[t * per:(t + 1) * per] = x.reshape(-1)
    allb = torch.empty(world * mx * per, dtype=dtype, device=device)
    dist.all_gather_into_tensor(allb, buf)
    out = []
    for r in range(world):
        for t in range(counts[r]):
            out.append(allb[(r * mx + t) * per:(r * mx + t + 1) * per].view(shape))
    return out


def _coll_tensor(t: torch.Tensor):
    """gloo (CPU tests, or two ranks sharing one GPU) reduces host tensors; NCCL device tensors."""
    import torch.distributed as dist
    return t.cpu() if (t.is_cuda and dist.get_backend() == "gloo") else t


def allreduce_sum_(t: torch.Tensor) -> torch.Tensor:
    """In-place exact u64 sum over the ranks (int64 two's-complement add = u64 add)."""
    import torch.distributed as dist
    h = _coll_tensor(t)
    dist.all_reduce(h, op=dist.ReduceOp.SUM)
    if h is not t:
        t.copy_(h)
    return t


def allgather_cts(params: blb.Params, local: list, counts: list, level: int) -> list:
    """All-gather ciphertexts (rank r holds counts[r] of them, in rank order) onto every rank."""
    import torch.distributed as dist
    like = torch.empty(2 * (level + 1) * params.N, dtype=torch.int64, device="cuda")
    items = [c.data.reshape(-1) for c in local]
    if dist.get_backend() == "gloo":
        items = [x.cpu() for x in items]
        like = like.cpu()
    full = allgather_ragged(items, counts, like=like)
    scales = [None] * len(counts)
    dist.all_gather_object(scales, [c.scale for c in local])   # per-output scales (exact doubles)
    flat = [x for r in scales for x in r]
    out = []
    for x, sc in zip(full, flat):
        out.append(blb.Ciphertext(x.to("cuda").reshape(2, level + 1, params.N).contiguous(), level, sc))
    return out


class FusedLinearLayer:
    def __init__(self, params: blb.Params, dims: Dims = BERT_BASE, rank: int = 0, world: int = 1,
                 bsgs: dict | None = None, level: int | None = None):
        self.p, self.dims, self.rank, self.world = params, dims, rank, world
        self.level = params.K - 1 if level is None else level
        b = dict(BSGS, **(bsgs or {}))
        L, d, H, ffn = dims.L, dims.d, dims.H, dims.ffn
        cm = blb.mhp_column_map(d, H, L, params.log_n)
        self.Hp = 1 << (H - 1).bit_length()
        qkv_map = cm + [d + c if c >= 0 else -1 for c in cm] + list(range(2 * d, 3 * d))
        self.n_mhp = len(cm) // (params.n // L)   # ciphertexts of Q (and of K)
        c = params.n // L

        def win(B: int):
            """this rank's baby-step window of [0, B) (None: one rank, the whole plan)"""
            if world == 1:
                return None
            if world > B:
                raise ValueError("%d ranks exceed the BSGS baby-step count B = %d" % (world, B))
            return shard(B, rank, world)

        self.plans = {
            "qkv": blb.MatmulPlan(params, L, d, 3 * d, col_map=qkv_map, bsgs_B=b["qkv"], level=self.level,
                                  window=win(min(b["qkv"], c))),
            "oproj": blb.MatmulPlan(params, L, self.Hp * (d // H), d, packing=blb.PACK_DIAGONAL, heads=self.Hp,
                                    bsgs_B=b["oproj"], level=self.level - 3, window=win(min(b["oproj"], c))),
            "ffn1": blb.MatmulPlan(params, L, d, ffn, bsgs_B=b["ffn1"], level=self.level,
                                   window=win(min(b["ffn1"], c))),
            "ffn2": blb.MatmulPlan(params, L, ffn, d, bsgs_B=b["ffn2"], level=self.level,
                                   window=win(min(b["ffn2"], c))),
        }
        # output ownership: rank r finishes (giant steps, ModDown, rescale) and masks a contiguous slice
        self.slices = {k: shard(pl.n_out, rank, world) for k, pl in self.plans.items()}
        g = params.n // (L * self.Hp)
        B_qk = b["qk"] or g
        # Q K^T consumes the 2 J MHP outputs of QKV at level-1 (row a7); Softmax x V (row f1) has inner
        # dimension L (V zero-padded d_h -> L); both sharded by baby-index window like the ct-pt plans
        self.qk = blb.QKPlan(params, L, H, d // H, bsgs_B=b["qk"], level=self.level - 1, window=win(B_qk))
        self.sv = blb.QKPlan(params, L, H, L, bsgs_B=b["qk"], level=self.level, window=win(B_qk))
        self.slices["qk"] = shard(self.qk.n_out, rank, world)
        self.slices["sv"] = shard(self.sv.n_out, rank, world)
        for name, n in [(k, pl.n_out) for k, pl in self.plans.items()] + [("qk", self.qk.n_out)]:
            if n > MAX_OUT:
                raise ValueError("%s: %d output ciphertexts exceed the mask-id range" % (name, n))
        self.pts, self.ws, self.outs = {}, None, {}
        self.pre_ct_pt = None   # optional hook(name) run right before each ct-pt MatMul (model.GPT2Stack)
        self.acc = None
        self.seq = 0      # inference counter: enters every mask id (fresh masks per step)

    # ---- setup (row a0) ----
    def rotation_steps(self) -> list[int]:
        s = set(self.qk.rotation_steps()) | set(self.sv.rotation_steps())
        for pl in self.plans.values():
            s.update(pl.rotation_steps())
        return sorted(s)

    def load_weights(self, WQ, WK, WV, WO, W1, W2):
        Wqkv = np.concatenate([WQ, WK, WV], axis=1)
        # MHP row reorder of W_O for the padded-head diagonal input: zero rows for padded heads
        dh = self.dims.d // self.dims.H
        WOp = np.zeros((self.Hp * dh, WO.shape[1]))
        WOp[:WO.shape[0]] = WO
        WO = WOp
        for name, W in (("qkv", Wqkv), ("oproj", WO), ("ffn1", W1), ("ffn2", W2)):
            if self.world == 1:
                first, count = self.slices[name]
                self.pts[name] = self.plans[name].encode_weights(W, first, count)
            else:   # the window's plaintexts of every output
                self.pts[name] = self.plans[name].encode_weights(W)
        self.qk_masks = self.qk.encode_masks()
        self.sv_masks = self.sv.encode_masks()
        nbytes = max([pl.workspace_bytes(pl.n_out) for k, pl in self.plans.items()] +
                     [self.qk.workspace_bytes(), self.sv.workspace_bytes()])
        self.ws = torch.empty(nbytes // 8 + 1, dtype=torch.int64, device="cuda")
        if self.world > 1:
            n_acc = max([pl.acc_numel() for pl in self.plans.values()] + [self.qk.acc_numel(), self.sv.acc_numel()])
            self.acc = torch.empty(n_acc, dtype=torch.int64, device="cuda")
        for k, pl in self.plans.items():
            self.outs[k] = [blb.Ciphertext.empty(self.p, self.level - 1) for _ in range(self.slices[k][1])]
        self.outs["qk"] = [blb.Ciphertext.empty(self.p, self.level - 4) for _ in range(self.qk.n_out)]
        self.outs["sv"] = [blb.Ciphertext.empty(self.p, self.level - 3) for _ in range(self.sv.n_out)]
        self.sv_dense = [blb.Ciphertext.empty(self.p, self.level - 3) for _ in range(self.sv.n_out // 2)]

    def plaintext_bytes(self) -> int:
        return (sum(int(t.numel()) * 8 for t in self.pts.values()) + int(self.qk_masks.numel()) * 8 +
                int(self.sv_masks.numel()) * 8)

    def n_plaintexts(self) -> int:
        if self.world > 1:
            return sum(self.plans[k].pt_count() for k in self.plans)
        return sum(self.plans[k].pt_count(*self.slices[k]) for k in self.plans)

    def mask_counts(self, name: str) -> list[int]:
        """Number of masked outputs of a block on every rank (for the end-of-layer all-gather)."""
        out = []
        for r in range(self.world):
            n = self.qk.n_out if name == "qk" else self.plans[name].n_out
            f, c = shard(n, r, self.world)
            lo = 2 * self.n_mhp if name == "qkv" else 0
            out.append(len([o for o in range(f, f + c) if o >= lo]))
        return out

    def mask_outputs(self, name: str) -> list[int]:
        """Plan output indices of the masked outputs of this rank."""
        first, count = self.slices[name]
        outs = range(first, first + count)
        if name == "qkv":   # only V is converted here; Q, K feed Q K^T (row a7)
            outs = [o for o in outs if o >= 2 * self.n_mhp]
        return list(outs)

    def mask_ids(self, name: str, seq: int) -> list[int]:
        """Global mask object ids of this rank's masked outputs in inference seq (C4, C19)."""
        return [mask_id(seq, name, o) for o in self.mask_outputs(name)]

    # ---- the hot path ----
    def ct_pt(self, keys: blb.Keys, name: str, src: list) -> list:
        """One ct-pt MatMul -> this rank's output slice (world 1: the fused single call)."""
        pl = self.plans[name]
        first, count = self.slices[name]
        if self.world == 1:
            return pl(keys, src, self.pts[name], first, count, ws=self.ws, outs=self.outs[name])
        n = pl.acc_numel()
        acc = pl.acc(keys, src, self.pts[name], acc_out=self.acc[:n], ws=self.ws)
        allreduce_sum_(acc)
        per = pl.acc_numel(1)
        return pl.finish(keys, acc[first * per:(first + count) * per], first, count, src[0].scale, ws=self.ws,
                         outs=self.outs[name][:count])

    def ct_ct(self, keys: blb.Keys, plan: blb.QKPlan, masks, Q: list, K: list, outs: list, name: str) -> list:
        """One ct-ct MatMul (C13) -> this rank's output slice (world 1: all outputs)."""
        if self.world == 1:
            return plan(keys, Q, K, masks, ws=self.ws, outs=outs)
        n = plan.acc_numel()
        acc = plan.acc(keys, Q, K, masks, acc_out=self.acc[:n], ws=self.ws)
        allreduce_sum_(acc)
        first, count = self.slices[name]
        a0, na = plan.acc_range(first, count)
        per = n // max(1, plan.acc_range(0, plan.n_out)[1])
        return plan.finish(keys, acc[a0 * per:(a0 + na) * per], first, count, Q[0].scale, K[0].scale, ws=self.ws,
                           outs=outs[first:first + count])

    def gather_qk_operands(self, outs: list):
        """Q and K ciphertexts (QKV outputs 0 .. 2J-1) on every rank."""
        if self.world == 1:
            return outs[:2 * self.n_mhp]
        counts = [shard(self.plans["qkv"].n_out, r, self.world)[1] for r in range(self.world)]
        full = allgather_cts(self.p, outs, counts, self.level - 1)
        return full[:2 * self.n_mhp]

    def softmax_v(self, keys: blb.Keys, S_cts: list, Vt_cts: list) -> list:
        """Row f1: S_h (x) Vpad_h by the ct-ct protocol, then the dense-diagonal collapse."""
        outs = self.ct_ct(keys, self.sv, self.sv_masks, S_cts, Vt_cts, self.outs["sv"], "sv")
        if self.world > 1:   # the out-projection consumes every collapsed diagonal
            counts = [shard(self.sv.n_out, r, self.world)[1] for r in range(self.world)]
            outs = allgather_cts(self.p, outs, counts, self.level - 3)
        half = len(outs) // 2
        for o in range(half):
            blb.add_into(self.p, outs[o], outs[o + half], self.sv_dense[o])
        return self.sv_dense

    def step(self, keys: blb.Keys, inputs: dict, mask_key: bytes, seq: int | None = None) -> list:
        """inputs: {'qkv': [ct]*3, 'sv_s': [ct]*J', 'sv_v': [ct]*J', 'ffn1': [...], 'ffn2': [...]}
        -> [(name, first mask id, (masked, share))] per block, this rank's outputs.  seq: the inference
        number entering the mask ids (default: the layer's own counter, incremented per call, so masks
        are never reused)."""
        if seq is None:
            seq = self.seq
        self.seq = seq + 1
        res = []
        for name in ("qkv", "oproj", "ffn1", "ffn2"):
            first, count = self.slices[name]
            if count == 0 and self.world == 1:
                continue
            src = self.softmax_v(keys, inputs["sv_s"], inputs["sv_v"]) if name == "oproj" else inputs[name]
            if self.pre_ct_pt is not None:
                self.pre_ct_pt(name)
            outs = self.ct_pt(keys, name, src)
            if name == "qkv":
                qk_in = self.gather_qk_operands(outs)
                J = self.n_mhp
                qk_out = self.ct_ct(keys, self.qk, self.qk_masks, qk_in[:J], qk_in[J:2 * J], self.outs["qk"], "qk")
                qf, qc = self.slices["qk"]
                if qc:
                    ids = self.mask_ids("qk", seq)
                    mine = qk_out if self.world > 1 else qk_out[qf:qf + qc]
                    res.append(("qk", ids[0], blb.ckks_to_mpc(self.p, mine, mask_key, ids[0])))
            ids = self.mask_ids(name, seq)
            if not ids:
                continue
            sel = [outs[o - first] for o in self.mask_outputs(name)]
            # ids of one block are contiguous: one mask launch per block
            res.append((name, ids[0], blb.ckks_to_mpc(self.p, sel, mask_key, ids[0])))
        return res


class LayerPipeline:
    """Host-to-host serving loop over one FusedLinearLayer (the e2e path of bench.py).

    Every step copies that step's encrypted inputs from pinned host memory to the device and reads
    the masked outputs + server shares back into pinned host memory.  Uploads and downloads run on
    two streams of their own (one per copy direction: on a single copy stream the upload of step k+1
    queued behind the download of step k, which waits for step k's evaluation, so every upload was
    exposed) and the inputs are double-buffered: the upload of step k+1 and the download of step k-1
    overlap the evaluation of step k on the compute stream; the only exposed transfers are the first
    upload and the last download.
    """

    def __init__(self, layer: FusedLinearLayer, keys: blb.Keys, mask_key: bytes, like_inputs: dict):
        self.layer, self.keys, self.mask_key = layer, keys, mask_key
        self.up, self.down = torch.cuda.Stream(), torch.cuda.Stream()
        # two device input sets (ping-pong), each a dict like the inputs of FusedLinearLayer.step
        self.dev = [{k: [blb.Ciphertext(torch.empty_like(c.data), c.level, c.scale) for c in v]
                     for k, v in like_inputs.items()} for _ in range(2)]
        self.free = [torch.cuda.Event() for _ in range(2)]      # compute done with input set s
        self.ready = [torch.cuda.Event() for _ in range(2)]     # upload into set s done
        self.host_out = [None, None]
        self.k = 0

    def submit(self, host_inputs: dict, gather=None, seq: int | None = None) -> list:
        """Enqueue one step; returns the pinned host buffers its results land in (valid after sync)."""
        s = self.k % 2
        comp = torch.cuda.current_stream()
        with torch.cuda.stream(self.up):
            if self.k >= 2:
                self.up.wait_event(self.free[s])
            for name, hs in host_inputs.items():
                for h, c in zip(hs, self.dev[s][name]):
                    c.data.copy_(h, non_blocking=True)
            self.ready[s].record(self.up)
        comp.wait_event(self.ready[s])
        res = self.layer.step(self.keys, self.dev[s], self.mask_key, seq)
        if gather is not None:
            res = gather(res)
        self.free[s].record(comp)
        tensors = []
        for r in res:
            tensors.extend(r[2] if isinstance(r[2], (tuple, list)) else (r[2],))
        if self.host_out[s] is None or len(self.host_out[s]) != len(tensors):
            self.host_out[s] = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in tensors]
        done = torch.cuda.Event()
        done.record(comp)
        with torch.cuda.stream(self.down):
            self.down.wait_event(done)
            for h, t in zip(self.host_out[s], tensors):
                if t.is_cuda:  # (results gathered over gloo on a shared GPU are host tensors already)
                    t.record_stream(self.down)
                h.copy_(t, non_blocking=True)
        self.k += 1
        return self.host_out[s]

    def drain(self, stream=None):
        """Make the caller's stream wait for every outstanding copy."""
        st = stream or torch.cuda.current_stream()
        st.wait_stream(self.up)
        st.wait_stream(self.down)
