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
config 3).  Work is sharded by output ciphertext (section 8(e)): rank r owns a
contiguous slice of every plan's outputs, holds only the plaintexts of that
slice, recomputes the (replicated) baby steps, and the masked results are
all-gathered at the end of the layer.  The BSGS split is fixed independently of
the number of ranks, so outputs are bit-identical at every GPU count.
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
BSGS = {"qkv": 64, "oproj": 16, "ffn1": 64, "ffn2": 16, "qk": 0}
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
        self.plans = {
            "qkv": blb.MatmulPlan(params, L, d, 3 * d, col_map=qkv_map, bsgs_B=b["qkv"], level=self.level),
            "oproj": blb.MatmulPlan(params, L, self.Hp * (d // H), d, packing=blb.PACK_DIAGONAL, heads=self.Hp,
                                    bsgs_B=b["oproj"], level=self.level - 3),
            "ffn1": blb.MatmulPlan(params, L, d, ffn, bsgs_B=b["ffn1"], level=self.level),
            "ffn2": blb.MatmulPlan(params, L, ffn, d, bsgs_B=b["ffn2"], level=self.level),
        }
        self.slices = {k: shard(pl.n_out, rank, world) for k, pl in self.plans.items()}
        # Q K^T consumes the 2 J MHP outputs of QKV at level-1 (row a7); with more than one
        # rank the Q / K ciphertexts are all-gathered first and Q K^T is replicated (its
        # outputs are masked by their owner only) -- see DESIGN.md section 8.
        self.qk = blb.QKPlan(params, L, H, d // H, bsgs_B=b["qk"], level=self.level - 1)
        self.slices["qk"] = shard(self.qk.n_out, rank, world)
        # Softmax x V (row f1): inner dimension L (V zero-padded d_h -> L), replicated like Q K^T
        self.sv = blb.QKPlan(params, L, H, L, bsgs_B=b["qk"], level=self.level)
        for name, n in [(k, pl.n_out) for k, pl in self.plans.items()] + [("qk", self.qk.n_out)]:
            if n > MAX_OUT:
                raise ValueError("%s: %d output ciphertexts exceed the mask-id range" % (name, n))
        self.pts, self.ws, self.outs = {}, None, {}
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
            first, count = self.slices[name]
            self.pts[name] = self.plans[name].encode_weights(W, first, count)
        self.qk_masks = self.qk.encode_masks()
        self.sv_masks = self.sv.encode_masks()
        nbytes = max([pl.workspace_bytes(self.slices[k][1]) for k, pl in self.plans.items()] +
                     [self.qk.workspace_bytes(), self.sv.workspace_bytes()])
        self.ws = torch.empty(nbytes // 8 + 1, dtype=torch.int64, device="cuda")
        for k, pl in self.plans.items():
            self.outs[k] = [blb.Ciphertext.empty(self.p, self.level - 1) for _ in range(self.slices[k][1])]
        self.qkv_full = [blb.Ciphertext.empty(self.p, self.level - 1) for _ in range(2 * self.n_mhp)]
        self.outs["qk"] = [blb.Ciphertext.empty(self.p, self.level - 4) for _ in range(self.qk.n_out)]
        self.outs["sv"] = [blb.Ciphertext.empty(self.p, self.level - 3) for _ in range(self.sv.n_out)]
        self.sv_dense = [blb.Ciphertext.empty(self.p, self.level - 3) for _ in range(self.sv.n_out // 2)]

    def plaintext_bytes(self) -> int:
        return (sum(int(t.numel()) * 8 for t in self.pts.values()) + int(self.qk_masks.numel()) * 8 +
                int(self.sv_masks.numel()) * 8)

    def n_plaintexts(self) -> int:
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
    def gather_qk_operands(self, outs: list):
        """Q and K ciphertexts (QKV outputs 0 .. 2J-1) on every rank."""
        if self.world == 1:
            return outs[:2 * self.n_mhp]
        counts = [shard(self.plans["qkv"].n_out, r, self.world)[1] for r in range(self.world)]
        full = allgather_ragged([o.data for o in outs], counts, like=self.qkv_full[0].data)
        scale = outs[0].scale if outs else 2.0 ** bi_log_delta()
        for g in range(2 * self.n_mhp):
            self.qkv_full[g].data.copy_(full[g])
            self.qkv_full[g].scale = scale
        return self.qkv_full

    def softmax_v(self, keys: blb.Keys, S_cts: list, Vt_cts: list) -> list:
        """Row f1: S_h (x) Vpad_h by the ct-ct protocol, then the dense-diagonal collapse."""
        outs = self.sv(keys, S_cts, Vt_cts, self.sv_masks, ws=self.ws, outs=self.outs["sv"])
        half = len(outs) // 2
        for o in range(half):
            blb.add_into(self.p, outs[o], outs[o + half], self.sv_dense[o])
        return self.sv_dense

    def step(self, keys: blb.Keys, inputs: dict, mask_key: bytes, seq: int | None = None) -> list:
        """inputs: {'qkv': [ct]*3, 'sv_s': [ct]*J', 'sv_v': [ct]*J', 'ffn1': [...], 'ffn2': [...]}
        -> [(name, first mask id, (masked, share))] per block.  seq: the inference number entering the
        mask ids (default: the layer's own counter, incremented per call, so masks are never reused)."""
        if seq is None:
            seq = self.seq
        self.seq = seq + 1
        res = []
        for name in ("qkv", "oproj", "ffn1", "ffn2"):
            first, count = self.slices[name]
            if count == 0 and not (name == "qkv" and self.world > 1):
                continue
            src = self.softmax_v(keys, inputs["sv_s"], inputs["sv_v"]) if name == "oproj" else inputs[name]
            outs = self.plans[name](keys, src, self.pts[name], first, count, ws=self.ws,
                                    outs=self.outs[name]) if count else []
            if name == "qkv":
                qk_in = self.gather_qk_operands(outs)
                J = self.n_mhp
                qk_out = self.qk(keys, qk_in[:J], qk_in[J:2 * J], self.qk_masks, ws=self.ws, outs=self.outs["qk"])
                qf, qc = self.slices["qk"]
                if qc:
                    ids = self.mask_ids("qk", seq)
                    res.append(("qk", ids[0], blb.ckks_to_mpc(self.p, qk_out[qf:qf + qc], mask_key, ids[0])))
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
                t.record_stream(self.down)
                h.copy_(t, non_blocking=True)
        self.k += 1
        return self.host_out[s]

    def drain(self, stream=None):
        """Make the caller's stream wait for every outstanding copy."""
        st = stream or torch.cuda.current_stream()
        st.wait_stream(self.up)
        st.wait_stream(self.down)
