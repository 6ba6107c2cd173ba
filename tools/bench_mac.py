"""ct-pt MatMul kernel breakdown on the BERT-base QKV plan (config 2, N = 2^16):
live CUDA-event times of the MAC, NTT and key-switch inner-product kernels for
one blb_ct_pt_matmul call.  Plaintexts are uniform random residues (encode is
row a0; values do not change the work).  MAC variants: env BLB_MAC_VARIANT.

    python tools/bench_mac.py [--plan qkv|oproj|ffn1|ffn2] [--iters 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import blb_inputs as bi  # noqa: E402
import paper_2508_19525_b200 as blb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--plan", default="qkv")
    ap.add_argument("--iters", type=int, default=5)
    args = ap.parse_args()
    g = blb.Params.from_preset(bi.BERT)
    L, d, H, ffn = 128, 768, 12, 3072
    if args.plan == "qkv":
        cm = blb.mhp_column_map(d, H, L, 16)
        qkv_map = cm + [d + c if c >= 0 else -1 for c in cm] + list(range(2 * d, 3 * d))
        plan = blb.MatmulPlan(g, L, d, 3 * d, col_map=qkv_map, bsgs_B=32, level=4)
    elif args.plan == "oproj":
        plan = blb.MatmulPlan(g, L, d, d, packing=blb.PACK_DIAGONAL, heads=H, bsgs_B=16, level=4)
    elif args.plan == "ffn1":
        plan = blb.MatmulPlan(g, L, d, ffn, bsgs_B=32, level=4)
    else:
        plan = blb.MatmulPlan(g, L, ffn, d, bsgs_B=8, level=4)
    keys, sk = blb.keygen(g, bi.crypto_key(1, 1), plan.rotation_steps())
    k = 5
    pts = torch.randint(0, 2 ** 39, (plan.n_pt, k, g.N), dtype=torch.int64, device="cuda")
    cts = [blb.Ciphertext(torch.randint(0, 2 ** 39, (2, k, g.N), dtype=torch.int64, device="cuda"), 4, 2.0 ** 40)
           for _ in range(plan.n_in)]
    ws = plan.workspace()
    outs = plan(keys, cts, pts, ws=ws)
    torch.cuda.synchronize()
    blb.timing_reset()
    blb.timing_enable(True)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.iters):
        plan(keys, cts, pts, ws=ws, outs=outs)
    e1.record(st)
    torch.cuda.synchronize()
    blb.timing_enable(False)
    tot = e0.elapsed_time(e1) / args.iters
    res = {"plan": args.plan, "variant": os.environ.get("BLB_MAC_VARIANT", "0"), "ms_per_call": tot}
    for name, cat in (("mac", 0), ("ntt", 1), ("ks_inner", 2)):
        r = blb.timing_read(cat)
        res[name] = {"ms_per_call": r["ms"] / args.iters, "alg_GBps": r["alg_bytes"] / (r["ms"] * 1e-3) / 1e9}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
