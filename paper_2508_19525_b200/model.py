"""Config 5 (BASELINE.json): GPT2-base, 12 layers of the fused-linear CKKS path on one rank group.

GPT2-base has the BERT-base layer shape (d = 768, 12 heads, FFN 3072; L = 128 tokens as
BASELINE.json sets it, the paper ran 64, reading S25), so every layer is one
layer.FusedLinearLayer step (QKV + Q K^T + masks, Softmax x V + W_O + mask, FFN1 + mask,
FFN2 + mask) with its own weights.  Its packed plaintexts are 56.7 GB per layer -- 680 GB for
12 layers, far beyond one B200's 180 GB.  Three storage modes (`mode`):
* "resident": every layer's packed plaintexts stay on the device (e.g. 1/8 per rank at world 8:
  85 GB for all 12 layers) -- no per-layer work;
* "coeffs" (the 1-GPU default): every layer's weights are kept as their compact, prime-independent
  encode -- the rounded integer coefficients of each plaintext, 5 bytes each
  (blb_matmul_encode_coeffs: 9.8 GB per layer, 118 GB for 12) -- and right before each ct-pt
  MatMul its plaintexts are expanded on the device (residues mod q_0..q_l, NTT, packed layout:
  blb_matmul_coeffs_to_pts) into ONE buffer shared by the four MatMuls (17 GB);
* "reencode": float64 weights resident (57 MB per layer), each layer re-encoded from them
  (slot build, double-double inverse embedding, rounding, NTT, packing) before its step.
Synthetic weights: SURVEY 8(d) config 5, seeds 100 + 10 * layer + m.
"""
from __future__ import annotations

import numpy as np
import torch

import paper_2508_19525_b200 as blb
from paper_2508_19525_b200.layer import Dims, FusedLinearLayer


def gpt2_layer_weights(layer: int, dims: Dims) -> list:
    """W_Q, W_K, W_V, W_O, W_1, W_2 of one layer: N(0, 0.04^2) (W_2: N(0, 0.02^2)), seeds 100 + 10 l + m."""
    d, f = dims.d, dims.ffn
    shapes = [(d, d), (d, d), (d, d), (d, d), (d, f), (f, d)]
    stds = [0.04, 0.04, 0.04, 0.04, 0.04, 0.02]
    return [np.random.default_rng(100 + 10 * layer + m).normal(0.0, sd, sh) for m, (sh, sd) in
            enumerate(zip(shapes, stds))]


class GPT2Stack:
    def __init__(self, params: blb.Params, n_layers: int = 12, dims: Dims = Dims(), bsgs: dict | None = None,
                 rank: int = 0, world: int = 1, resident: bool | None = None, budget_bytes: float = 120e9,
                 mode: str | None = None):
        """mode: "resident" / "coeffs" / "reencode" (module docstring); None picks resident when this
        rank's packed plaintexts of all layers fit budget_bytes, else coeffs when the compact
        coefficients fit it, else reencode.  resident=True/False is the older spelling of
        mode="resident" / the default non-resident mode."""
        self.p, self.n_layers, self.dims = params, n_layers, dims
        self.layer = FusedLinearLayer(params, dims, rank, world, bsgs=bsgs)
        self.w_dev = []      # per layer: device float64 matrices in the plans' shapes
        self.pts = []        # resident mode: per layer the encoded plaintexts
        self.coefs = []      # coeffs mode: per layer the compact coefficients of every plan
        for l in range(n_layers):
            WQ, WK, WV, WO, W1, W2 = gpt2_layer_weights(l, dims)
            Wqkv = np.concatenate([WQ, WK, WV], axis=1)
            dh = dims.d // dims.H
            WOp = np.zeros((self.layer.Hp * dh, WO.shape[1]))
            WOp[:WO.shape[0]] = WO
            self.w_dev.append({k: torch.tensor(np.ascontiguousarray(w), dtype=torch.float64, device="cuda")
                               for k, w in (("qkv", Wqkv), ("oproj", WOp), ("ffn1", W1), ("ffn2", W2))})
        # first layer through the layer's own loader: allocates the plaintext buffers, masks, workspace
        self.layer.load_weights(*gpt2_layer_weights(0, dims))
        self.loaded = 0
        per_layer = sum(int(t.numel()) * 8 for t in self.layer.pts.values())
        coef_layer = sum(self._coef_bytes(name) for name in self.layer.plans)
        if mode is None:
            if resident is not None:
                mode = "resident" if resident else "coeffs"
            elif per_layer * n_layers <= budget_bytes:
                mode = "resident"
            else:
                mode = "coeffs" if coef_layer * n_layers <= budget_bytes else "reencode"
        self.mode = mode
        self.resident = mode == "resident"
        if mode == "resident":
            for l in range(n_layers):
                self.pts.append({k: self._encode(l, k) for k in self.layer.plans})
        elif mode == "coeffs":
            # one plaintext buffer shared by the four MatMuls (the largest plan's size)
            big = max(int(t.numel()) for t in self.layer.pts.values())
            shared = torch.empty(big, dtype=torch.int64, device="cuda")
            self.layer.pts = {k: shared[:int(t.numel())] for k, t in self.layer.pts.items()}
            torch.cuda.empty_cache()
            for l in range(n_layers):
                self.coefs.append({k: self._slice_call(k, "encode_coeffs", self.w_dev[l][k]) for k in self.layer.plans})
            self.layer.pre_ct_pt = self._expand
            self.loaded = -1

    def _slice_call(self, name: str, method: str, arg, out=None):
        pl = self.layer.plans[name]
        if self.layer.world == 1:
            first, count = self.layer.slices[name]
            return getattr(pl, method)(arg, first, count, out=out)
        return getattr(pl, method)(arg, out=out)

    def _coef_bytes(self, name: str) -> int:
        pl = self.layer.plans[name]
        first, count = self.layer.slices[name] if self.layer.world == 1 else (0, pl.n_out)
        return pl.pt_count(first, count) * 5 * self.p.N

    def _encode(self, l: int, name: str, out=None) -> torch.Tensor:
        return self._slice_call(name, "encode_weights", self.w_dev[l][name], out=out)

    def _expand(self, name: str):
        """coeffs mode, right before the ct-pt MatMul `name` of the loaded layer."""
        self._slice_call(name, "coeffs_to_pts", self.coefs[self.loaded][name], out=self.layer.pts[name])

    def load_layer(self, l: int):
        """Make layer l's plaintexts the ones the layer step streams."""
        if self.mode == "resident":
            self.layer.pts = self.pts[l]
        elif self.mode == "reencode" and self.loaded != l:
            for name in self.layer.plans:
                self._encode(l, name, out=self.layer.pts[name])
        self.loaded = l

    def rotation_steps(self) -> list[int]:
        return self.layer.rotation_steps()

    def step(self, keys: blb.Keys, inputs: list, mask_key: bytes, seq0: int | None = None) -> list:
        """inputs[l]: the client's fresh ciphertexts of layer l (dict as FusedLinearLayer.step).
        -> per layer the masked outputs + server shares (the client reconstructs, runs the MPC
        nonlinear layers and re-encrypts the next layer's inputs)."""
        out = []
        seq = self.layer.seq if seq0 is None else seq0
        for l in range(self.n_layers):
            self.load_layer(l)
            out.append(self.layer.step(keys, inputs[l % len(inputs)], mask_key, seq=seq + l))
        return out
