"""Per-block device time of the benched BERT-base layer step (diagnostic; not a bench line).

Builds the same FusedLinearLayer as bench.py and wraps its block calls (ct-pt MatMuls by name, the
ct-ct Q.K^T, Softmax.V, the masks) in CUDA events on the launching stream; prints ms per block,
averaged over --steps after --warmup steps.

    python tools/block_times.py [--steps 5] [--warmup 2]
"""
import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import blb_inputs as bi  # noqa: E402
import paper_2508_19525_b200 as blb  # noqa: E402
from paper_2508_19525_b200 import packing  # noqa: E402
from paper_2508_19525_b200.layer import Dims, FusedLinearLayer  # noqa: E402

BSGS = dict(bi.BENCH_BSGS)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--bsgs", default="", help='JSON overrides of the BSGS dict, e.g. {"qkv": 32}')
    ap.add_argument("--only", default="", choices=["", "sv", "qk"],
                    help="run only Softmax.V (sv) or Q.K^T (qk), one call inside the NVTX range 'only' "
                         "(for an ncu launch list of that block)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    dims = dict(L=128, d=768, H=12, ffn=3072)
    preset = bi.BERT
    params = blb.Params.from_preset(preset, device=0)
    bsgs = dict(BSGS, **(json.loads(args.bsgs) if args.bsgs else {}))
    layer = FusedLinearLayer(params, Dims(**dims), 0, 1, bsgs=bsgs)
    A = bi.bert_attention_inputs(dims["L"], dims["d"])
    F = bi.bert_ffn_inputs(dims["L"], dims["d"], dims["H"], dims["ffn"])
    keys, sk = blb.keygen(params, A["keys_key"], layer.rotation_steps(), relin=True)
    layer.load_weights(A["WQ"], A["WK"], A["WV"], F["WO"], F["W1"], F["W2"])
    delta = 2.0 ** preset.log_delta
    sv_s, sv_v = packing.softmax_v_operands(F["S"], F["V"], params.n)
    slots = {"qkv": packing.spatial_slots(A["X"], params.n), "sv_s": sv_s, "sv_v": sv_v,
             "ffn1": packing.spatial_slots(F["X2"], params.n), "ffn2": packing.spatial_slots(F["H1"], params.n)}
    inputs, cid = {}, 0
    for name, zs in slots.items():
        pts = params.encode(torch.tensor(zs), delta, layer.level)
        inputs[name] = [blb.encrypt(params, sk, pts[b], layer.level, A["enc_key"], 4096 + (cid := cid + 1), delta)
                        for b in range(zs.shape[0])]
    del sk
    times = collections.defaultdict(list)
    recording = [False]

    def wrap(obj, attr, label_fn):
        fn = getattr(obj, attr)

        def inner(*a, **kw):
            if not recording[0]:
                return fn(*a, **kw)
            st = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            r = fn(*a, **kw)
            e1.record(st)
            times[label_fn(a)].append((e0, e1))
            return r
        setattr(obj, attr, inner)

    wrap(layer, "ct_pt", lambda a: "ct_pt:" + a[1])
    wrap(layer, "ct_ct", lambda a: "ct_ct:" + a[-1])
    wrap(blb, "ckks_to_mpc", lambda a: "masks")
    orig_sv = layer.softmax_v

    def sv(*a, **kw):  # Softmax.V (ct-ct with its collapse) excluding the out-proj ct-pt
        if not recording[0]:
            return orig_sv(*a, **kw)
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        recording[0] = False
        r = orig_sv(*a, **kw)
        recording[0] = True
        e1.record(st)
        times["softmax_v (ct-ct + collapse)"].append((e0, e1))
        return r
    layer.softmax_v = sv
    if args.only:
        if args.only == "sv":
            call = lambda: orig_sv(keys, inputs["sv_s"], inputs["sv_v"])  # noqa: E731
        else:
            outs = layer.ct_pt(keys, "qkv", inputs["qkv"])
            qk_in = layer.gather_qk_operands(outs)
            J = layer.n_mhp
            call = lambda: layer.ct_ct(keys, layer.qk, layer.qk_masks, qk_in[:J], qk_in[J:2 * J],  # noqa: E731
                                       layer.outs["qk"], "qk")
        for _ in range(args.warmup):
            call()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("only")
        call()
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        return
    for _ in range(args.warmup):
        layer.step(keys, inputs, A["mask_key"])
    torch.cuda.synchronize()
    recording[0] = True
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        layer.step(keys, inputs, A["mask_key"])
    e1.record()
    torch.cuda.synchronize()
    out = {k: sum(a.elapsed_time(b) for a, b in v) / args.steps for k, v in times.items()}
    out["step_total"] = e0.elapsed_time(e1) / args.steps
    out = {k: round(v, 3) for k, v in out.items()}
    out["bsgs"] = bsgs
    print(json.dumps(out))


if __name__ == "__main__":
    main()
