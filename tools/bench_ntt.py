"""NTT throughput microbenchmark (row a1): limb transforms per second for several batch sizes,
through the C ABI of a given libblb.so build (SURVEY 8(d) metric 2).

    python tools/bench_ntt.py [--lib path/to/libblb.so] [--rows 64,320,960] [--logn 16] [--prime i]
    python tools/bench_ntt.py --sweep      # N = 2^12, 2^14, 2^15, 2^16 x batches {1, 2k, 2(k+a)b, KS batch}
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
    ap.add_argument("--logn", type=int, default=16)
    ap.add_argument("--sweep", action="store_true")
    args = ap.parse_args()
    if args.sweep:
        # batches: 1 limb, 2k = 10 (a ciphertext), 2 (k + alpha) beta = 60 (one key switch's extended
        # digits), and a 128-job key-switch batch's ModUp rows (128 x 25 = 3200 -> 3198 = 533 x 6)
        for logn in (12, 14, 15, 16):
            for prime, rows in ((1, "1"), (0, "1"), (-1, "12,60,3198")):
                args.logn, args.prime, args.rows = logn, prime, rows
                run(args)
        return
    run(args)


def run(args):
    L = ctypes.CDLL(args.lib)
    vp = ctypes.c_void_p
    L.blb_params_create.argtypes = [vp, ctypes.c_int, vp, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.blb_prime_chain.argtypes = [ctypes.c_int, vp, ctypes.c_int, vp]
    L.blb_ntt.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.c_int, vp]
    L.blb_intt.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.c_int, vp]
    P = bi.BERT
    bits = list(P.q_bits) + list(P.p_bits)
    pr = (ctypes.c_uint64 * 6)()
    assert L.blb_prime_chain(args.logn, (ctypes.c_int * 6)(*bits), 6, pr) == 0
    h = ctypes.c_void_p()
    qa = (ctypes.c_uint64 * 5)(*pr[:5])
    pa = (ctypes.c_uint64 * 1)(pr[5])
    assert L.blb_params_create(ctypes.byref(h), args.logn, qa, 5, pa, 1, 5, 0) == 0
    N = 1 << args.logn
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
    print(json.dumps({"lib": os.path.basename(args.lib), "logN": args.logn,
                      "prime": "mixed (6 chain primes)" if args.prime < 0 else args.prime, "results": res}))


if __name__ == "__main__":
    main()
