#!/usr/bin/env python
"""bench.py -- ms per BERT-base layer of BLB's fused-linear CKKS evaluation on B200.

Metric (BASELINE.json): "ms per BERT-base layer fused-linear CKKS eval; NTT
limbs/s and HBM GB/s fraction".  One step = one pass of the whole hot path over
one layer's synthetic inputs: QKV ct-pt MatMul (C11, MHP) + out-projection
(C12, diagonal input) + FFN1 + FFN2, every MatMul with hoisted baby-step
rotations, MAC, giant-step key switches and rescale, the ct-ct MatMul Q_h K_h^T
for all heads (row a7: MHP + BSGS, relinearisation), then the CKKS->MPC masks
(server half of Alg. 1) of every converted output, and Softmax x V (row f1) with
its dense-diagonal collapse feeding the out-projection.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun (one rank per GPU, NCCL; bench.py --gpus N spawns it when run
directly): every MatMul is sharded by BSGS baby-step window, the partial accumulators are
summed exactly by one NCCL all-reduce, each output's owner finishes and masks it, and the
masked results are all-gathered.
"""
from __future__ import annotations

import argparse
import itertools
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import blb_inputs as bi  # noqa: E402

METRIC = "ms per BERT-base layer fused-linear CKKS eval"
# BSGS baby-step counts B per MatMul (C11, plan parameter S15); shared by both arms and by the
# full-size parity tests (tests/test_gpu_bert.py imports the same dict)
BSGS = dict(bi.BENCH_BSGS)
UNIT = "ms"
FALLBACK_HBM = 6650.0


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# --------------------------------------------------------------------------- clocks
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.index = index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                smax.append(float(r[1]))
                for nm, v in zip(names, r[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        os.unlink(self.f.name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- oracle (CPU baseline)
def cpu_info() -> dict:
    model = "?"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count() or 1}


def set_omp_threads(n: int):
    """OpenMP threads of the oracle's C library for the calling thread's next parallel regions."""
    import ctypes
    import ctypes.util
    name = ctypes.util.find_library("gomp") or "libgomp.so.1"
    ctypes.CDLL(name).omp_set_num_threads(int(n))


def layer_counts(dims) -> dict:
    """Slice-equivalents of one layer step from the oracle's own plans (C11 / C12 / C13):
    key switches (rotations + relinearisations), ct-pt products, ModDown+rescales, tensor products,
    masks -- the same schedule the GPU step runs (launch counters in the bench line agree)."""
    import oracle.matmul as mm
    import oracle.matmul_cc as cc
    n = bi.BERT.n
    L, d, H, ffn = dims["L"], dims["d"], dims["H"], dims["ffn"]
    cm = mm.mhp_column_map(d, H, L, n)
    qkv_map = cm + [d + c if c >= 0 else -1 for c in cm] + list(range(2 * d, 3 * d))
    Hp = 1 << (H - 1).bit_length()
    plans = [mm.plan_spatial(np.ones((d, 3 * d)), L, n, BSGS["qkv"], col_map=qkv_map),
             mm.plan_diagonal(np.ones((Hp * (d // H), d)), Hp, L, n, BSGS["oproj"]),
             mm.plan_spatial(np.ones((d, ffn)), L, n, BSGS["ffn1"]),
             mm.plan_spatial(np.ones((ffn, d)), L, n, BSGS["ffn2"])]
    c = {"ks": sum(p.n_rotations for p in plans), "prod": sum(p.n_plaintexts for p in plans),
         "mdr": sum(p.n_out for p in plans), "tensor": 0, "mask": sum(p.n_out for p in plans)}
    for qk in (cc.plan_qk(L, H, d // H, n), cc.plan_sv(L, H, n)):
        qc = qk.counts()
        acc3 = qk.accumulators()
        c["ks"] += qc["rotations"] + qc["relin"]
        c["prod"] += qk.J * qk.B * (2 * qk.g - 1) + 2 * qk.J * (qk.G - 1) + sum(
            1 for (u, w, f) in acc3 for i in range(qk.B) if qk.mask3(u, i, w, f).any())
        c["tensor"] += qc["cmult"]
        c["mdr"] += qk.J * (qk.B + qk.G) + qk.G * qk.B + len(acc3)
    qk0 = cc.plan_qk(L, H, d // H, n)
    c["mask"] += qk0.n_out - 2 * qk0.J       # Q, K outputs of QKV feed Q K^T; its diagonals are masked
    return c


def oracle_slice(threads: int, preset=bi.BERT) -> dict:
    """The CPU oracle, as it stands, on one stated slice of the layer at N = 2^16, level 4 (k = 5),
    timed directly: one baby-step rotation (hoisted-form ModUp + key switch + ModDown, C8), one
    (b', g) unit of the FFN1 MAC (3 inputs x B = 64 = 192 ct-pt products summed, C11), its giant
    step kept in Q u P + the fused ModDown/rescale (C11 lazy giant sum, C17), one ct-ct (u, i)
    stage of Q K^T (J = 4 tensor products summed + relinearisation in Q u P + ModDown/rescale,
    C13), and one CKKS->MPC mask (C14).  Plaintext / key values do not change the work, so uniform
    residues stand in for encoded weights and keys (encode is row a0)."""
    import oracle as O
    set_omp_threads(threads)
    P = preset
    primes = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    ctx = O.Ctx(P.log_n, primes[:5], primes[5:], P.dnum)
    rng = np.random.default_rng(0)
    lvl, k = 4, 5

    def rnd(polys, limbs):
        return np.stack([np.stack([rng.integers(0, ctx.mods[i], ctx.N, dtype=np.uint64) for i in limbs])
                         for _ in range(polys)])

    ct = O.Ct(rnd(2, range(k)), lvl, 2.0 ** 40)
    g = ctx.galois(128)
    key = np.stack([rnd(2, range(len(primes))) for _ in range(ctx.beta_top)])
    keys = O.Keys(None, None, {g: key, ctx.galois(64 * 128): key}, key)
    n_prod = 3 * BSGS["ffn1"]
    pts = [rnd(1, range(k))[0] for _ in range(n_prod)]
    ct3 = O.Ct(rnd(2, range(4)), 3, 2.0 ** 40)
    t = {}
    t0 = time.perf_counter()
    O.rotate(ctx, ct, keys, 128)
    t1 = time.perf_counter()
    acc = O.mul_pt(ctx, ct, pts[0], 1.0)
    for p in pts[1:]:
        acc = O.add(ctx, acc, O.mul_pt(ctx, ct, p, 1.0))
    t2 = time.perf_counter()
    ye = O.rotate_ext(ctx, acc, keys, 64 * 128)
    t3 = time.perf_counter()
    y = O.moddown_rescale(ctx, ye)
    t4 = time.perf_counter()
    dsum = None
    for _ in range(4):
        tt = O.tensor(ctx, ct3, ct3)
        dsum = tt if dsum is None else O.add(ctx, dsum, tt)
    t5 = time.perf_counter()
    O.moddown_rescale(ctx, O.relinearize_ext(ctx, dsum, keys))
    t6 = time.perf_counter()
    O.mask(ctx, y, bytes(32), 0)
    t7 = time.perf_counter()
    t = {"rotation": t1 - t0, "prod": (t2 - t1) / n_prod, "rotate_ext": t3 - t2, "mdr": t4 - t3,
         "tensor": (t5 - t4) / 4, "relin_ext+mdr": t6 - t5, "mask": t7 - t6}
    return {"ms": 1e3 * (t7 - t0), "per_op_s": t, "threads": threads}


def slice_desc() -> str:
    return ("oracle (u128 C + __float128, OpenMP) at N=2^16, k=5, directly timed per slice: 1 baby-step rotation "
            "(ModUp + key switch + ModDown) + one FFN1 (b',g) MAC unit (192 ct-pt products) + its giant step in Q u P "
            "with the fused ModDown/rescale + one Q.K^T (u,i) stage (4 tensor products + relinearisation + "
            "ModDown/rescale) + 1 CKKS->MPC mask")


def layer_estimate_ms(per_op: dict, counts: dict) -> float:
    """Layer-equivalent of the timed slice: each timed operation kind times its count in one layer
    step (every key switch at the full rotation's cost: an upper bound for the hoisted ones)."""
    return 1e3 * (counts["ks"] * per_op["rotation"] + counts["prod"] * per_op["prod"] +
                  counts["mdr"] * per_op["mdr"] + counts["tensor"] * per_op["tensor"] +
                  counts["mask"] * per_op["mask"])


def cpu_baseline(dims, preset=bi.BERT) -> dict:
    """The oracle timed on the host: the slice at 1 thread and at all cores (bounded, ~10-30 s)."""
    info = cpu_info()
    allc = info["nproc"]
    oracle_slice(allc, preset)               # warm: library load, table build
    ra = oracle_slice(allc, preset)
    r1 = oracle_slice(1, preset)
    counts = layer_counts(dims)
    return {"value": ra["ms"], "unit": "ms per slice", "cores": allc, "kind": "oracle", "sample": slice_desc(),
            "ms_per_slice_1thread": r1["ms"], "cpu_model": info["cpu_model"], "nproc": info["nproc"],
            "per_op_s_all_cores": ra["per_op_s"], "per_op_s_1thread": r1["per_op_s"],
            "layer_counts": counts,
            "ms_per_layer_est_all_cores": layer_estimate_ms(ra["per_op_s"], counts),
            "ms_per_layer_est_1thread": layer_estimate_ms(r1["per_op_s"], counts),
            "estimate_how": "sum over operation kinds of (directly timed op time x its count per layer step)"}


def run_reference(args, dims, preset=bi.BERT):
    """--impl reference: the oracle timed on host cores (all of them), each step one slice of the
    layer (oracle_slice).  ms_per_step is the timed slice; value is its layer-equivalent in the
    metric's unit (each timed operation times its count per layer step, stated in the line)."""
    info = cpu_info()
    counts = layer_counts(dims)
    oracle_slice(info["nproc"], preset)       # warm-up outside the timed steps (library load, tables)
    steps, ests = [], []
    for s in range(args.warmup + args.steps):
        r = oracle_slice(info["nproc"], preset)
        if s >= args.warmup:
            steps.append(r["ms"])
            ests.append(layer_estimate_ms(r["per_op_s"], counts))
    ms_step = float(np.median(steps))
    v = float(np.median(ests))
    line = {"impl": "reference", "metric": metric_name(dims), "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": config_dict(dims, args.gpus, preset),
            "timed_region": "each step = one directly timed oracle slice (ms_per_step); value = that slice's "
                            "layer-equivalent (layer_counts x per-op times)",
            "layer_counts": counts,
            "cpu_baseline": {"kind": "oracle", "value": v, "unit": UNIT, "cores": info["nproc"],
                             "cpu_model": info["cpu_model"], "sample": slice_desc(), "ms_per_slice": ms_step},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def model_name(dims):
    return "BERT-base" if dims["d"] == 768 else "BERT-large"


def metric_name(dims):
    return METRIC.replace("BERT-base", model_name(dims))


def preset_desc(preset) -> str:
    def fmt(bits):
        return ",".join("%dx%d" % (b, n) if n > 1 else str(b)
                        for b, n in ((b, len(list(g))) for b, g in itertools.groupby(bits)))
    return "N=2^%d, Q={%s}, P={%s}, dnum=%d" % (preset.log_n, fmt(preset.q_bits), fmt(preset.p_bits), preset.dnum)


def config_dict(dims, world, preset=bi.BERT):
    return {"workload": model_name(dims) + " layer fused-linear CKKS (config 2 QKV + Q.K^T, Softmax.V + out-proj, config 3 "
                        "FFN1/FFN2, CKKS->MPC masks), " + preset_desc(preset) +
                        ("" if preset is bi.BERT else " (the config-2 dnum=1 variant, reading C23)"),
            "L": dims["L"], "d": dims["d"], "heads": dims["H"], "ffn": dims["ffn"], "log_n": preset.log_n,
            "limbs": len(preset.q_bits), "special_primes": len(preset.p_bits), "dnum": preset.dnum,
            "bsgs": dict(BSGS),
            "layer_ops": ["qkv_ct_pt(MHP)", "qk_ct_ct(MHP+BSGS)", "mask(QK^T)", "mask(V)",
                          "softmaxV_ct_ct(pad+collapse)", "oproj_diag_ct_pt(level 1)", "mask", "ffn1_ct_pt", "mask",
                          "ffn2_ct_pt", "mask"],
            "not_included": "non-MatMul HE ops of Table 6 blocks 2-5 (row f2) and the MPC protocols",
            "l2": "inputs larger than L2 (%s of plaintexts streamed per step)" % ("~57 GB" if dims["d"] == 768 else "~91 GB"),
            "parallelism": ("dp%d: every MatMul sharded by BSGS baby-step window, exact NCCL all-reduce of the "
                            "partial accumulators, owners finish + mask their output ciphertexts, NCCL all-gathers "
                            "(Q/K, Softmax.V outputs, masked results)" % world) if world > 1 else "dp1"}


def ntt_pipes(ctr: dict, ntt: dict, params, pipes: dict, steps: int) -> dict:
    """The NTT's arithmetic-pipe fraction next to its HBM fraction: algorithmic
    ops per butterfly -- 60-bit rows (integer kernel, truncated-quotient Shoup): 9 IMAD-class
    multiplies (3 for the quotient, 3 + 3 for the two low 64-bit products); 40-bit rows (FP64
    kernel): 8 FP64 ops (DMUL, 3 DFMA, 2 DADD in the product, DADD + DSUB in the butterfly) --
    times the measured pipe peaks, against the live NTT time."""
    if not ntt["ms"]:
        return {}
    bfly = (params.N // 2) * params.log_n
    n_all, n_int = ctr["limb_ntts"], ctr.get("limb_ntts_int", 0)
    t_int = n_int * bfly * 9 / pipes["imad_per_s"]
    t_f64 = (n_all - n_int) * bfly * 8 / pipes["dfma_per_s"]
    t = ntt["ms"] * 1e-3
    return {"rows_int_per_step": n_int / steps, "rows_fp64_per_step": (n_all - n_int) / steps,
            "pipe_peaks": pipes, "pipe_bound_ms_per_step": 1e3 * (t_int + t_f64) / steps,
            "pipe_frac": (t_int + t_f64) / t,
            "pipe_frac_how": "(int rows x 9 IMAD + FP64 rows x 8 FP64 ops per butterfly) at the measured peaks, "
                             "the two pipes taken one after the other, / live NTT time",
            "hbm_frac": ntt["alg_bytes"] / t / 1e9 / float(measured_peaks().get("hbm_gbs", FALLBACK_HBM))}


def run_gpt2(args, rank: int, world: int, local: int):
    """Config 5: GPT2-base, 12 layers (d 768, 12 heads, FFN 3072, L = 128), each layer one fused-linear
    step with its own weights; the 680 GB of per-layer plaintexts do not fit one GPU, so (model.GPT2Stack
    mode "coeffs") every layer's weights stay resident as compact 5-byte integer coefficients and each
    MatMul's plaintexts are expanded on the device (residues, NTT, packing) right before it -- timed: it is
    per-inference work at 1 GPU ("reencode": the older full re-encode from float64 weights).
    One step = 12 layers."""
    import torch
    import torch.distributed as dist

    import paper_2508_19525_b200 as blb
    from paper_2508_19525_b200 import packing
    from paper_2508_19525_b200.layer import Dims
    from paper_2508_19525_b200.model import GPT2Stack
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dims = Dims(**bi.GPT2_BASE)
    params = blb.Params.from_preset(bi.BERT, device=local)
    t0 = time.perf_counter()
    stack = GPT2Stack(params, 12, dims, bsgs=BSGS, rank=rank, world=world, mode=args.gpt2_mode)
    keys, sk = blb.keygen(params, bi.crypto_key(4, 5), stack.rotation_steps(), relin=True)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    A = bi.bert_attention_inputs(dims.L, dims.d, config_id=5)
    F = bi.bert_ffn_inputs(dims.L, dims.d, dims.H, dims.ffn, config_id=5)
    sv_s, sv_v = packing.softmax_v_operands(F["S"], F["V"], params.n)
    slots = {"qkv": packing.spatial_slots(A["X"], params.n), "sv_s": sv_s, "sv_v": sv_v,
             "ffn1": packing.spatial_slots(F["X2"], params.n), "ffn2": packing.spatial_slots(F["H1"], params.n)}
    inputs, cid = {}, 0
    for name, zs in slots.items():
        pts = params.encode(torch.tensor(zs), 2.0 ** 40, stack.layer.level)
        inputs[name] = [blb.encrypt(params, sk, pts[b], stack.layer.level, A["enc_key"], 9000 + cid + b, 2.0 ** 40)
                        for b in range(zs.shape[0])]
        cid += zs.shape[0]
    del sk
    for _ in range(args.warmup):
        stack.step(keys, [inputs], A["mask_key"])
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    blb.reset_counters()
    e0.record(st)
    for _ in range(args.steps):
        stack.step(keys, [inputs], A["mask_key"])
    e1.record(st)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ctr = blb.counters()
    if rank == 0:
        print(json.dumps({
            "metric": "ms per GPT2-base 12-layer fused-linear CKKS eval (config 5)", "value": ms, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded N(0,1) activations, N(0,0.04^2) weights, seeds 100 + 10 layer + m)",
            "config": {"workload": "GPT2-base 12 layers, L=128, d=768, 12 heads, FFN 3072; per layer the fused-linear "
                                   "step of the BERT-base bench; N=2^16, Q={60,40x4}, P={60}, dnum=5",
                       "plaintexts": {
                           "resident": "resident (this rank's share of all 12 layers fits)",
                           "coeffs": "680 GB of packed plaintexts for 12 layers exceed one GPU: the weights stay "
                                     "resident as 5-byte rounded encode coefficients (118 GB for 12 layers) and each "
                                     "MatMul's plaintexts are expanded on the device (residues, NTT, packing) right "
                                     "before it, inside the timed step",
                           "reencode": "re-encoded on the device per layer from resident float64 weights (680 GB of "
                                       "packed plaintexts for 12 layers exceed one GPU)"}[stack.mode],
                       "gpt2_mode": stack.mode,
                       "bsgs": dict(BSGS), "parallelism": "dp%d" % world},
            "gpu_launches": ctr["launches"], "counters_per_step": {k: v / args.steps for k, v in ctr.items()},
            "clocks": clk, "setup_s": t_setup}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def f2_blocks(dims, args, device: int) -> dict:
    """Row f2 for one layer (reading C21): per layer 12 negExp chains (Softmax exp of H x L x L),
    12 Softmax smul_cc, 2 LayerNorm heads and 2 tails (L x d: d / (n / L) ciphertexts each) and the
    GeLU head over L x ffn, on fresh ciphertexts of the Table-6 block-3 preset (N = 2^15, RNS
    {60, 40 x 7} + {60}, scale 2^40).  Timed like the main step: W warm-ups, K steps between CUDA
    events on the launching stream."""
    import torch

    import paper_2508_19525_b200 as blb
    from paper_2508_19525_b200.blocks import Chains
    P = bi.F2
    params = blb.Params.from_preset(P, device=device)
    n, L = params.n, dims["L"]
    c = n // L
    ch = Chains(params, None)
    keys, sk = blb.keygen(params, bi.crypto_key(4, 200), ch.rotation_steps(L), relin=True)
    ch.keys = keys
    rng = np.random.default_rng(200)
    top = params.K - 1
    delta = 2.0 ** P.log_delta
    cid = [0]

    def enc(z, lvl=top):
        cid[0] += 1
        return blb.encrypt(params, sk, params.encode(torch.tensor(z)[None], delta, lvl)[0], lvl,
                           bi.crypto_key(5, 200), cid[0], delta)

    n_sm = -(-dims["H"] * L * L // n)
    n_ln = -(-dims["d"] // c)
    n_ge = -(-dims["ffn"] // c)
    sm = [(enc(rng.uniform(-6, 0, n)), enc(rng.uniform(0, 7, n))) for _ in range(n_sm)]
    sm_inv = [(enc(rng.uniform(0, 1, n)), enc(rng.uniform(0.01, 1, n))) for _ in range(n_sm)]
    ln = [enc(rng.normal(0, 1, n)) for _ in range(n_ln)]
    xmu = [enc(rng.normal(0, 1, n)) for _ in range(n_ln)]
    rs = enc(rng.uniform(0.5, 2, n))
    gam = [rng.normal(1, 0.1, n) for _ in range(n_ln)]
    bet = [rng.normal(0, 0.1, n) for _ in range(n_ln)]
    ge = [enc(rng.uniform(-2.7, 2.7, n)) for _ in range(n_ge)]
    del sk

    parts = ["negexp", "smul", "ln_head", "ln_tail", "gelu_head"]
    evs = {p: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for p in parts}
    acc_ms = {p: 0.0 for p in parts}

    def step(timed=False):
        st_ = torch.cuda.current_stream()

        def mark(p, i):
            if timed:
                evs[p][i].record(st_)
        mark("negexp", 0)
        ch.negexp_n([x for x, _ in sm], [xb for _, xb in sm])             # block 2 (depth 7)
        mark("negexp", 1)
        mark("smul", 0)
        ch.muls([xe for xe, _ in sm_inv], [r for _, r in sm_inv])         # Softmax smul_cc (block 3 head)
        mark("smul", 1)
        mark("ln_head", 0)
        for _ in range(2):
            ch.ln_head(ln, L, dims["d"])               # blocks 3 and 5 tails: LayerNorm lines 1-6
        mark("ln_head", 1)
        mark("ln_tail", 0)
        for _ in range(2):
            ch.ln_tail(xmu, rs, gam, bet)              # blocks 4 and 1 heads: LayerNorm lines 8-10
        mark("ln_tail", 1)
        mark("gelu_head", 0)
        ch.gelu_head_n(ge, bi.GELU_COEF)               # block 4: GeLU lines 1-4
        mark("gelu_head", 1)
        if timed:
            torch.cuda.synchronize()
            for p in parts:
                acc_ms[p] += evs[p][0].elapsed_time(evs[p][1])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("f2_steps")
    e0.record(st)
    for _ in range(args.steps):
        step()
    e1.record(st)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    step(timed=True)   # one more step with per-chain events (the breakdown, not the headline)
    return {"ms_per_step": e0.elapsed_time(e1) / args.steps, "breakdown_ms": acc_ms,
            "preset": "N=2^15, Q={60,40x7}, P={60}, dnum=8 "
            "(Table 6 block 3, P:719)", "ciphertexts": {"negexp": n_sm, "smul": n_sm, "layernorm": n_ln,
                                                      "gelu": n_ge}}


# --------------------------------------------------------------------------- our arm
TOY_METRIC = "ms per config-1 toy step (ct-pt MatMul 16x16x16 + CKKS->MPC mask)"


def toy_oracle_step(threads: int) -> float:
    """The whole config-1 step in the oracle (no extrapolation): MatMul of the encrypted X with W
    (C11, B = 16) and the CKKS->MPC mask of the output.  -> seconds."""
    import oracle as O
    import oracle.matmul as mm
    set_omp_threads(threads)
    P, d = bi.TOY, bi.toy_inputs()
    primes = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    ctx = O.Ctx(P.log_n, primes[:3], primes[3:], P.dnum)
    plan = mm.plan_spatial(d["W"], 16, ctx.n, 16)
    keys = O.keygen(ctx, d["keys_key"], plan.rotation_steps())
    delta = 2.0 ** P.log_delta
    cts = [O.encrypt(ctx, d["enc_key"], keys.s_ntt, O.encode(ctx, z, delta, ctx.K - 1), ctx.K - 1, t, delta)
           for t, z in enumerate(mm.pack_spatial(d["X"], ctx.n))]
    t0 = time.perf_counter()
    (y,) = mm.matmul_cp(ctx, keys, cts, plan)
    O.mask(ctx, y, d["mask_key"], 0)
    return time.perf_counter() - t0


def run_toy(args):
    """BASELINE config 1: N = 2^12, Q = {60, 40, 40}, P = {60}, dnum = 3; X in R^{16x16} ~ U(-1, 1)
    (seed 1), W ~ U(-1/2, 1/2) (seed 2); one step = the ct-pt MatMul (15 baby + 1 giant rotation,
    31 plaintexts, fused ModDown + rescale) + the CKKS->MPC mask of its output.  Launch-latency bound
    at this size (a handful of microsecond kernels); reported for completeness of the config list."""
    info = cpu_info()
    if args.impl == "reference":
        toy_oracle_step(info["nproc"])
        ts = [toy_oracle_step(info["nproc"]) for _ in range(args.warmup + args.steps)][args.warmup:]
        v = 1e3 * float(np.median(ts))
        print(json.dumps({"impl": "reference", "metric": TOY_METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False,
                          "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                          "config": {"workload": "config 1 toy: " + preset_desc(bi.TOY) + ", X W 16x16x16 + mask"},
                          "cpu_baseline": {"kind": "oracle", "value": v, "unit": UNIT, "cores": info["nproc"],
                                           "cpu_model": info["cpu_model"], "sample": "the whole toy step"},
                          "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
              flush=True)
        return
    import torch
    import paper_2508_19525_b200 as blb
    from paper_2508_19525_b200 import packing
    P, d = bi.TOY, bi.toy_inputs()
    params = blb.Params.from_preset(P)
    plan = blb.MatmulPlan(params, 16, 16, 16, bsgs_B=16)
    keys, sk = blb.keygen(params, d["keys_key"], plan.rotation_steps())
    pts = plan.encode_weights(d["W"])
    delta = 2.0 ** P.log_delta
    zs = packing.spatial_slots(d["X"], params.n)
    cts = [blb.encrypt(params, sk, params.encode(torch.tensor(z), delta, params.K - 1), params.K - 1, d["enc_key"],
                       t, delta) for t, z in enumerate(zs)]
    stream = torch.cuda.current_stream()

    def step(inp, seq):
        out = plan(keys, inp, pts)
        return blb.ckks_to_mpc(params, out, d["mask_key"], seq)

    for s in range(args.warmup):
        step(cts, s)
    torch.cuda.synchronize()
    blb.reset_counters()
    blb.timing_reset()
    blb.timing_enable(True)
    clocks = Clocks(0)
    clocks.start()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for s in range(args.steps):
        step(cts, 1000 + s)
    ev1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    blb.timing_enable(False)
    ms = ev0.elapsed_time(ev1) / args.steps
    ctr = blb.counters()
    mac = blb.timing_read(blb.TIMING_MAC)
    # e2e: input ciphertexts from pinned host memory, masked output + share back to pinned memory
    host_in = [c.data.cpu().pin_memory() for c in cts]
    dev_in = [torch.empty_like(c.data) for c in cts]
    host_m = torch.empty(2 * params.N, dtype=torch.int64).pin_memory()
    host_s = torch.empty(params.N, dtype=torch.int64).pin_memory()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s in range(args.steps):
        for h, dv in zip(host_in, dev_in):
            dv.copy_(h, non_blocking=True)
        m, sh = step([blb.Ciphertext(dv, c.level, c.scale) for dv, c in zip(dev_in, cts)], 2000 + s)
        host_m.copy_(m.reshape(-1), non_blocking=True)
        host_s.copy_(sh.reshape(-1), non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    peaks = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", FALLBACK_HBM))
    mac_gbs = mac["alg_bytes"] / (mac["ms"] * 1e-3) / 1e9 if mac["ms"] > 0 else None
    line = {"metric": TOY_METRIC, "value": ms, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (X ~ U(-1,1) seed 1, W ~ U(-1/2,1/2) seed 2)",
            "config": {"workload": "config 1 toy: " + preset_desc(P) + ", X W 16x16x16 + CKKS->MPC mask",
                       "bsgs_B": 16, "plaintexts": plan.n_pt, "rotations": plan.n_rotations,
                       "l2": "working set (< 2 MB) is L2-resident: a latency-bound configuration"},
            "roofline": {"kernel": "k_mac_tma4 + k_mac_q0 (ct-pt weight MAC: packed limbs + the q0 limb, concurrent)", "bound": "hbm", "achieved": mac_gbs,
                         "peak": hbm_peak, "unit": "GB/s", "frac": mac_gbs / hbm_peak if mac_gbs else None,
                         "traffic": None, "note": "31 plaintexts of 2^12 coefficients: launch latency, not HBM"},
            "gpu_launches": ctr["launches"], "counters_per_step": {k: v / args.steps for k, v in ctr.items()},
            "clocks": clk,
            "e2e": {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": int(sum(h.numel() * 8 for h in host_in)),
                    "d2h_bytes_per_step": int((host_m.numel() + host_s.numel()) * 8)}}
    if not args.no_cpu_baseline:
        toy_oracle_step(info["nproc"])
        ta = toy_oracle_step(info["nproc"])
        t1 = toy_oracle_step(1)
        line["cpu_baseline"] = {"value": 1e3 * ta, "unit": UNIT, "cores": info["nproc"], "kind": "oracle",
                                "sample": "the whole toy step (MatMul + mask), directly timed",
                                "ms_1thread": 1e3 * t1, "cpu_model": info["cpu_model"]}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-f2", action="store_true")
    ap.add_argument("--dims", default="base", choices=["base", "large"])
    ap.add_argument("--gpt2-mode", default=None, choices=[None, "resident", "coeffs", "reencode"],
                    help="config 5 plaintext storage (model.GPT2Stack; default: by memory budget)")
    ap.add_argument("--model", default="layer", choices=["layer", "gpt2"],
                    help="gpt2: config 5, the 12-layer GPT2-base stack with per-layer on-device re-encode")
    ap.add_argument("--preset", default="bert", choices=["bert", "bert_dnum1"],
                    help="bert_dnum1: the config-2 dnum = 1 variant (one digit, four special primes; C23)")
    ap.add_argument("--config", default="layer", choices=["layer", "toy"],
                    help="toy: BASELINE config 1 (N=2^12, ct-pt MatMul 16x16x16 + CKKS->MPC mask)")
    args = ap.parse_args()
    preset = {"bert": bi.BERT, "bert_dnum1": bi.BERT_DNUM1}[args.preset]
    dims = dict(L=128, d=768, H=12, ffn=3072) if args.dims == "base" else dict(L=128, d=1024, H=16, ffn=4096)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launched directly with --gpus N: spawn one rank per GPU (the driver launches through torchrun)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print("bench.py: --gpus %d but WORLD_SIZE=%d; using the launched world" % (args.gpus, world), file=sys.stderr)
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config == "toy":
        if rank == 0:
            run_toy(args)
        return
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, dims, preset)
        return

    import torch
    import torch.distributed as dist

    import paper_2508_19525_b200 as blb
    from paper_2508_19525_b200 import packing
    from paper_2508_19525_b200.layer import Dims, FusedLinearLayer

    if args.model == "gpt2":
        return run_gpt2(args, rank, world, local)

    ngpu = max(1, torch.cuda.device_count())
    shared_gpu = world > ngpu      # more ranks than GPUs: functional run of the multi-rank path only
    local = local % ngpu
    torch.cuda.set_device(local)
    if world > 1:
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    coll_dev = "cpu" if shared_gpu else "cuda"
    t_setup0 = time.perf_counter()
    params = blb.Params.from_preset(preset, device=local)
    layer = FusedLinearLayer(params, Dims(**dims), rank, world, bsgs=BSGS)
    A = bi.bert_attention_inputs(dims["L"], dims["d"])
    F = bi.bert_ffn_inputs(dims["L"], dims["d"], dims["H"], dims["ffn"])
    keys, sk = blb.keygen(params, A["keys_key"], layer.rotation_steps(), relin=True)
    torch.cuda.synchronize()
    t_keys = time.perf_counter() - t_setup0
    t0 = time.perf_counter()
    layer.load_weights(A["WQ"], A["WK"], A["WV"], F["WO"], F["W1"], F["W2"])
    torch.cuda.synchronize()
    t_encode = time.perf_counter() - t0

    # client-side inputs: encrypt once (fresh ciphertexts at the top level)
    delta = 2.0 ** preset.log_delta
    lvl = layer.level
    sv_s, sv_v = packing.softmax_v_operands(F["S"], F["V"], params.n)
    slots = {"qkv": packing.spatial_slots(A["X"], params.n), "sv_s": sv_s, "sv_v": sv_v,
             "ffn1": packing.spatial_slots(F["X2"], params.n), "ffn2": packing.spatial_slots(F["H1"], params.n)}
    inputs, cid = {}, 0
    for name, zs in slots.items():
        pts = params.encode(torch.tensor(zs), delta, lvl)
        inputs[name] = []
        for b in range(zs.shape[0]):
            inputs[name].append(blb.encrypt(params, sk, pts[b], lvl, A["enc_key"], 4096 + cid, delta))
            cid += 1
    del sk
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()

    from paper_2508_19525_b200.layer import allgather_ragged

    def gather(res):
        """End-of-layer exchange: every rank receives all masked outputs + server shares.  Every rank
        walks the same block list (a rank may own no masked output of a block)."""
        if world == 1:
            return res
        mine = {name: (id0, m, s) for name, id0, (m, s) in res}
        out = []
        for name in ("qk", "qkv", "oproj", "ffn1", "ffn2"):
            counts = layer.mask_counts(name)
            if sum(counts) == 0:
                continue
            id0, m, s = mine.get(name, (None, None, None))
            items = [] if m is None else [torch.cat([m[t].reshape(-1), s[t].reshape(-1)]).to(coll_dev)
                                          for t in range(m.shape[0])]
            out.append((name, id0, allgather_ragged(items, counts, like=torch.empty(3 * params.N, dtype=torch.int64,
                                                                                    device=coll_dev))))
        return out

    def step():
        return gather(layer.step(keys, inputs, A["mask_key"]))

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    pipes = blb.pipe_peaks(local)   # measured IMAD / DFMA peaks (NTT pipe-fraction denominators)
    # ---- timed region (device events; max over ranks) ----
    blb.reset_counters()
    blb.timing_reset()
    blb.timing_enable(True)
    clocks = Clocks(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    torch.cuda.nvtx.range_push("timed_steps")
    for _ in range(args.steps):
        step()
    torch.cuda.nvtx.range_pop()
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    blb.timing_enable(False)
    ms_total = ev0.elapsed_time(ev1)
    ctr = blb.counters()
    mac = blb.timing_read(blb.TIMING_MAC)
    ntt = blb.timing_read(blb.TIMING_NTT)
    ksi = blb.timing_read(blb.TIMING_KS_INNER)
    mmac = blb.timing_read(blb.TIMING_MASK_MAC)
    tsum = blb.timing_read(blb.TIMING_TENSOR)
    ms_step = ms_total / args.steps
    if world > 1:
        t = torch.tensor([ms_step], device=coll_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())

    # ---- e2e through the public API with host buffers (layer.LayerPipeline) ----
    # every step: H2D of that step's encrypted inputs from pinned memory and D2H of its masked
    # outputs + server shares into pinned memory, on a copy stream double-buffered against compute
    e2e = None
    if not args.no_e2e:
        from paper_2508_19525_b200.layer import LayerPipeline
        host_in = {k: [torch.empty_like(c.data, device="cpu").pin_memory() for c in v] for k, v in inputs.items()}
        for k, v in inputs.items():
            for h, c in zip(host_in[k], v):
                h.copy_(c.data)
        h2d = sum(h.numel() * h.element_size() for v in host_in.values() for h in v)
        pipe = LayerPipeline(layer, keys, A["mask_key"], inputs)
        for _ in range(2):  # warm-up (pinned output buffers, allocator)
            pipe.submit(host_in, gather)
        pipe.drain()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        pipe.up.wait_stream(stream)
        pipe.down.wait_stream(stream)
        d2h = 0
        for _ in range(args.steps):
            outs_host = pipe.submit(host_in, gather)
            d2h = sum(t.numel() * t.element_size() for t in outs_host)
        pipe.drain(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        e2e_ms = e0.elapsed_time(e1) / args.steps
        if world > 1:
            t = torch.tensor([e2e_ms], device=coll_dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "pipeline": "upload and download streams double-buffered against compute (layer.LayerPipeline)"}

    # ---- row f2: the fused-block chains between MPC steps (Table 6 block-3 preset, N = 2^15) ----
    f2 = None
    if rank == 0 and not args.no_f2:
        f2 = f2_blocks(dims, args, local)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", FALLBACK_HBM))
    mac_gbs = mac["alg_bytes"] / (mac["ms"] * 1e-3) / 1e9 if mac["ms"] > 0 else None
    traffic = None
    tf = os.path.join(ROOT, "profiles", "mac_traffic.json")
    if os.path.exists(tf):  # DRAM bytes / algorithmic bytes of one ncu --set full capture, scaled per launch
        try:
            traffic = json.load(open(tf))["ratio"] * mac["alg_bytes"] / max(1, mac["launches"])
        except Exception:
            traffic = None
    line = {
        "metric": metric_name(dims), "value": ms_step, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded N(0,1) activations, N(0,0.04^2) weights)",
        "config": config_dict(dims, world, preset),
        "roofline": {"kernel": "k_mac_tma4 + k_mac_q0 (ct-pt weight MAC, row a3: packed limbs + the q0 limb, concurrent)", "bound": "hbm", "achieved": mac_gbs, "peak": hbm_peak,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6.65 TB/s",
                     "unit": "GB/s", "frac": (mac_gbs / hbm_peak) if mac_gbs else None, "traffic": traffic,
                     "alg_bytes_per_launch": mac["alg_bytes"] / max(1, mac["launches"]),
                     "ms_per_launch": mac["ms"] / max(1, mac["launches"]),
                     "share_of_step": mac["ms"] / ms_total if ms_total else None},
        "ntt": {**ntt_pipes(ctr, ntt, params, pipes, args.steps),
                "limbs_per_s": (ntt["alg_bytes"] / (16.0 * params.N)) / (ntt["ms"] * 1e-3) if ntt["ms"] else None,
                "alg_gbs": ntt["alg_bytes"] / (ntt["ms"] * 1e-3) / 1e9 if ntt["ms"] else None,
                "share_of_step": ntt["ms"] / ms_total if ms_total else None, "launches": ntt["launches"]},
        "ks_inner": {"alg_gbs": ksi["alg_bytes"] / (ksi["ms"] * 1e-3) / 1e9 if ksi["ms"] else None,
                     "share_of_step": ksi["ms"] / ms_total if ms_total else None},
        "mask_mac": {"kernel": "k_mac_j / k_mac (ct-ct masks, rows a7/f1; bytes = mask + rotation tiles staged)",
                     "alg_gbs": mmac["alg_bytes"] / (mmac["ms"] * 1e-3) / 1e9 if mmac["ms"] else None,
                     "share_of_step": mmac["ms"] / ms_total if ms_total else None},
        "tensor_sum": {"kernel": "k_tensor_sum22 (ct-ct J-sum of tensor products, rows a7/f1)",
                       "alg_gbs": tsum["alg_bytes"] / (tsum["ms"] * 1e-3) / 1e9 if tsum["ms"] else None,
                       "share_of_step": tsum["ms"] / ms_total if ms_total else None},
        "gpu_launches": ctr["launches"],
        "counters_per_step": {k: v / args.steps for k, v in ctr.items()},
        "clocks": clk,
        "setup_s": {"keygen": t_keys, "weight_encode": t_encode, "plaintexts": layer.n_plaintexts(),
                    "plaintext_GB": layer.plaintext_bytes() / 1e9},
        "e2e": e2e,
        "shared_gpu": shared_gpu or None,   # true: ranks shared one GPU (functional check, not a scaling number)
        "full_layer": ({"ms": ms_step + f2["ms_per_step"], "matmul_blocks_ms": ms_step, "f2_chains_ms": f2["ms_per_step"],
                        "what": "the fused-linear MatMul step (value) + the row-f2 chains of one layer (negExp, "
                                "Softmax smul_cc, 2 x LayerNorm head/tail, GeLU head) on the Table-6 block-3 preset",
                        "f2": f2} if f2 else None),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(dims, preset)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
