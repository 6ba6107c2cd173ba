"""Measured lower bound for an int8-split tensor-core NTT pass (f4).

A 2^16 NTT as two 256-point passes is, per limb and pass, Y = T X with T the 256 x 256 twiddle
matrix of one prime and X the 256 x 256 limb (plus a pointwise twiddle between the passes).  Exact
residues need a byte split of both operands: 40-bit residues -> 5 signed bytes each, so Y = sum over
c = a + b of 2^(8c) Y_c with Y_c = sum_{a+b=c} T_b X_a -- 9 int8 GEMMs whose K concatenates the
(a, b) pairs (K = 256 x #pairs, int32 sums < 5 * 2^22), i.e. one 256 x 6400 x (256 * limbs) product;
60-bit residues need 8 x 8 = 64 slices (15 GEMMs, K total 256 x 64).  This times only those int8
products with cuBLASLt (torch._int_mm, the library GEMM, an upper bound on what a hand-written
tcgen05 kernel would reach) for a batch of limbs of one prime -- the slice recombination, the mod-q
reduction and the twiddle pass are NOT included -- and prints it beside the FP64 / integer NTT
kernels' time per pass for the same batch (tools/bench_ntt.py).

    python tools/bench_int8_ntt_gemm.py [--limbs 960]
"""
import argparse
import json
import os
import subprocess
import sys

import torch


def time_slices(limbs: int, nb: int, iters: int = 10, transposed: bool = False) -> dict:
    """nb bytes per residue: c = 0 .. 2 nb - 2 GEMMs with K = 256 * #pairs(c).  transposed: Y^T = X^T T^T
    (M = 256 * limbs, N = 256) instead of Y = T X (M = 256, N = 256 * limbs)."""
    n = 256 * limbs
    dev = "cuda"
    pairs = [sum(1 for a in range(nb) for b in range(nb) if a + b == c) for c in range(2 * nb - 1)]
    mm, nn = (n, 256) if transposed else (256, n)
    A = [torch.randint(-128, 128, (mm, 256 * p), dtype=torch.int8, device=dev) for p in pairs]
    # _int_mm wants the second operand column-major: allocate [N, K] and pass its transpose
    B = [torch.randint(-128, 128, (nn, 256 * p), dtype=torch.int8, device=dev).t() for p in pairs]
    for a, b in zip(A, B):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        for a, b in zip(A, B):
            torch._int_mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    ops = 2.0 * 256 * 256 * sum(pairs) * n
    return {"bytes_per_residue": nb, "gemms": len(pairs), "K_total": 256 * sum(pairs), "M": mm, "N": nn,
            "us_per_pass": us, "int8_tops": ops / (us * 1e-6) / 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--limbs", type=int, default=960)
    args = ap.parse_args()
    out = {"limbs": args.limbs, "nominal_int8_dense_tops": 4500,
           "int8_gemm_only": {"40-bit (5 x 5 slices)": [time_slices(args.limbs, 5, transposed=t) for t in (False, True)],
                              "60-bit (8 x 8 slices)": [time_slices(args.limbs, 8, transposed=t) for t in (False, True)]}}
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for prime, name in ((1, "fp64_kernel_40bit"), (0, "int_kernel_60bit")):
        r = subprocess.run([sys.executable, os.path.join(root, "tools", "bench_ntt.py"), "--rows", str(args.limbs),
                            "--prime", str(prime)], capture_output=True, text=True)
        res = json.loads(r.stdout.strip().splitlines()[-1])["results"]["ntt_%d" % args.limbs]
        out[name] = {"us_both_passes": res["us"], "us_per_pass": res["us"] / 2, "limbs_per_s": res["limbs_per_s"]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
