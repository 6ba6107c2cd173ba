"""NTT throughput microbenchmark (row a1): limb transforms per second at N = 2^16
for several batch sizes, through the C ABI of a given libblb.so build.

    python tools/bench_ntt.py [--lib path/to/libblb.so] [--rows 64,320,960]
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import blb_inputs as bi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2508_19525_b200", "libblb.so"))
    ap.add_argument("--rows", default="60,300,960,1920")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--prime", type=int, default=-1, help="run every row on this prime index (default: all six)")
    args = ap.parse_args()
    L = ctypes.CDLL(args.lib)
    vp = ctypes.c_void_p
    L.blb_params_create.argtypes = [vp, ctypes.c_int, vp, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.blb_prime_chain.argtypes = [ctypes.c_int, vp, ctypes.c_int, vp]
    L.blb_ntt.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.c_int, vp]
    L.blb_intt.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.c_int, vp]
    P = bi.BERT
    bits = list(P.q_bits) + list(P.p_bits)
    pr = (ctypes.c_uint64 * 6)()
    assert L.blb_prime_chain(P.log_n, (ctypes.c_int * 6)(*bits), 6, pr) == 0
    h = ctypes.c_void_p()
    qa = (ctypes.c_uint64 * 5)(*pr[:5])
    pa = (ctypes.c_uint64 * 1)(pr[5])
    assert L.blb_params_create(ctypes.byref(h), 16, qa, 5, pa, 1, 5, 0) == 0
    N = 1 << 16
    res = {}
    st = torch.cuda.current_stream()
    for rows in [int(r) for r in args.rows.split(",")]:
        nl = 6 if args.prime < 0 else 1
        polys = rows // nl
        data = torch.randint(0, 2 ** 39, (polys, nl, N), dtype=torch.int64, device="cuda")
        pidx = (ctypes.c_int32 * nl)(*(range(6) if args.prime < 0 else [args.prime]))
        for name, fn in (("ntt", L.blb_ntt), ("intt", L.blb_intt)):
            for _ in range(3):
                fn(h, ctypes.c_void_p(data.data_ptr()), pidx, nl, polys, ctypes.c_void_p(st.cuda_stream))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(args.iters):
                fn(h, ctypes.c_void_p(data.data_ptr()), pidx, nl, polys, ctypes.c_void_p(st.cuda_stream))
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.iters
            limbs = polys * nl
            res["%s_%d" % (name, limbs)] = {"us": ms * 1e3, "limbs_per_s": limbs / (ms * 1e-3),
                                            "alg_GBps": limbs * 16 * N / (ms * 1e-3) / 1e9}
    print(json.dumps({"lib": os.path.basename(args.lib), "results": res}))


if __name__ == "__main__":
    main()
