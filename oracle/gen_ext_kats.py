"""Known answers for the extended semantics (TEST INFRASTRUCTURE).

Writes tests/golden/ext_known_answers.json: small gemm_ext / conv2d_ext calls whose
expected outputs are computed here INDEPENDENTLY of oracle/ext_oracle.c and of the
GPU code — numpy matrix products on transposed views and a padded / strided /
dilated window formulation for conv — on inputs of small integers and binary
fractions, so every product and sum is exact and the answers can be checked by
hand (the first case of each kind is worked in the comments below).  Dispatch
failures are listed with the check the header names.

    python oracle/gen_ext_kats.py
"""
import json
import os

import numpy as np

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "ext_known_answers.json")


def gemm_case(name, ta, tb, m, n, k, lda, ldb, ldc, alpha, beta, A, B, C, f32=False):
    A, B, C = (np.asarray(x, dtype=np.float64) for x in (A, B, C))
    rA, cA = (k, m) if ta else (m, k)
    rB, cB = (n, k) if tb else (k, n)
    Am = np.lib.stride_tricks.as_strided(A, (rA, cA), (lda * 8, 8))
    Bm = np.lib.stride_tricks.as_strided(B, (rB, cB), (ldb * 8, 8))
    opA = Am.T if ta else Am
    opB = Bm.T if tb else Bm
    out = C.copy()
    prod = opA @ opB
    for i in range(m):
        for j in range(n):
            v = alpha * prod[i, j] if beta == 0 else alpha * prod[i, j] + beta * C[i * ldc + j]
            out[i * ldc + j] = float(np.float32(v)) if f32 else v
    return {"name": name, "spec": "gemm_ext", "sizes": [ta, tb, m, n, k, lda, ldb, ldc], "floats": [alpha, beta],
            "bufs": [A.tolist(), B.tolist(), [None if np.isnan(x) else x for x in C.tolist()]],
            "is_f32": [0, 0, int(f32)], "status": 0,
            "expect": [A.tolist(), B.tolist(), [None if np.isnan(x) else x for x in out.tolist()]]}


def conv_case(name, n, c, h, w, k, r, s, sh, sw, ph, pw, dh, dw, oh, ow, IN, WT, status=0, f32=False):
    IN = np.asarray(IN, dtype=np.float64).reshape(n, c, h, w)
    WT = np.asarray(WT, dtype=np.float64).reshape(k, c, r, s)
    case = {"name": name, "spec": "conv2d_ext", "sizes": [n, c, h, w, k, r, s, sh, sw, ph, pw, dh, dw, oh, ow],
            "floats": [], "is_f32": [0, 0, int(f32)], "status": status}
    out_len = n * k * max(oh, 1) * max(ow, 1)
    OUT0 = np.full(out_len, -7.0)
    case["bufs"] = [IN.ravel().tolist(), WT.ravel().tolist(), OUT0.tolist()]
    if status:
        case["expect"] = case["bufs"]
        return case
    P = np.pad(IN, ((0, 0), (0, 0), (ph, ph), (pw, pw)))  # zero padding
    out = np.zeros((n, k, oh, ow))
    for u in range(r):
        for v in range(s):
            win = P[:, :, u * dh: u * dh + sh * (oh - 1) + 1: sh, v * dw: v * dw + sw * (ow - 1) + 1: sw]
            out += np.einsum("nchw,kc->nkhw", win, WT[:, :, u, v])
    o = out.ravel()
    if f32:
        o = o.astype(np.float32).astype(np.float64)
    case["expect"] = [IN.ravel().tolist(), WT.ravel().tolist(), o.tolist()]
    return case


def main():
    cases = []
    # opA = A^T for A = [[1, 2], [3, 4]] (stored k x m, lda 2) = [[1, 3], [2, 4]]; B = I;
    # C = 2 * opA + 0.5 * 1 = [[2.5, 6.5], [4.5, 8.5]]
    cases.append(gemm_case("gemm_transA_alpha_beta", 1, 0, 2, 2, 2, 2, 2, 2, 2.0, 0.5, [1, 2, 3, 4], [1, 0, 0, 1],
                           [1, 1, 1, 1]))
    # transB, lda/ldc with gaps (the gaps of C keep their 7s), beta 0: NaN in C is not read
    cases.append(gemm_case("gemm_transB_gaps_beta0", 0, 1, 2, 3, 2, 3, 2, 4, 1.0, 0.0,
                           [1, 2, 99, 3, 4, 99], [1, 0.5, 2, 0.25, -1, 1],
                           [float("nan"), 7, 7, 7, 7, 7, 7, 7]))
    cases.append(gemm_case("gemm_both_trans", 1, 1, 3, 2, 2, 3, 2, 2, -1.0, 2.0, [1, 2, 3, 4, 5, 6],
                           [0.5, 1, 1.5, 2], [1, 1, 1, 1, 1, 1]))
    # exact in FP64 (dyadic, < 53 significant bits), not representable in f32: the
    # write-back rounding is visible
    e = 2.0 ** -30
    cases.append(gemm_case("gemm_f32_round", 0, 0, 1, 1, 3, 3, 1, 1, 1.0, 0.0, [1 + e, 2 + e, 3 + e], [1, 1, 1],
                           [0.0], f32=True))
    for nm, sizes, why in (("gemm_ldc_too_small", [0, 0, 2, 3, 2, 2, 3, 2], "leading dimension"),
                           ("gemm_bad_trans_flag", [2, 0, 2, 2, 2, 2, 2, 2], "transpose flag"),
                           ("gemm_footprint", [0, 0, 2, 2, 2, 2, 2, 2], "footprint")):
        c = {"name": nm, "spec": "gemm_ext", "sizes": sizes, "floats": [1.0, 0.0], "is_f32": [0, 0, 0],
             "status": 2, "why": why}
        lens = (4, 4, 4) if nm != "gemm_footprint" else (3, 4, 4)
        c["bufs"] = [[1.0] * lens[0], [1.0] * lens[1], [0.0] * lens[2]]
        c["expect"] = c["bufs"]
        cases.append(c)
    # stride 2: out[y, x] = in[2y, 2x] + in[2y+1, 2x+1] for in = 0..15 (4 x 4), w = I(2) -> [5, 9, 21, 25]
    cases.append(conv_case("conv_stride2", 1, 1, 4, 4, 1, 2, 2, 2, 2, 0, 0, 1, 1, 2, 2, range(16), [1, 0, 0, 1]))
    # pad 1 on a 3 x 3 image of ones, 3 x 3 kernel of ones: window counts [4,6,4,6,9,6,4,6,4]
    cases.append(conv_case("conv_pad1", 1, 1, 3, 3, 1, 3, 3, 1, 1, 1, 1, 1, 1, 3, 3, [1] * 9, [1] * 9))
    # dilation 2, 2 x 2 kernel of ones on 0..24 (5 x 5): 20y + 4x + 24 -> [24,28,32,44,48,52,64,68,72]
    cases.append(conv_case("conv_dil2", 1, 1, 5, 5, 1, 2, 2, 1, 1, 0, 0, 2, 2, 3, 3, range(25), [1] * 4))
    rng = np.random.default_rng(11)
    IN = rng.integers(-8, 9, 2 * 3 * 6 * 7) / 4.0
    WT = rng.integers(-8, 9, 2 * 3 * 3 * 2) / 8.0
    # n=2 c=3 h=6 w=7 k=2 r=3 s=2, stride (2,1), pad (1,0), dil (1,2): oh = (6+2-2-1)/2+1 = 3, ow = (7-2-1)/1+1 = 5
    cases.append(conv_case("conv_mixed", 2, 3, 6, 7, 2, 3, 2, 2, 1, 1, 0, 1, 2, 3, 5, IN, WT))
    cases.append(conv_case("conv_mixed_f32", 2, 3, 6, 7, 2, 3, 2, 2, 1, 1, 0, 1, 2, 3, 5, IN + 2.0 ** -30, WT,
                           f32=True))
    cases.append(conv_case("conv_oh_mismatch", 1, 1, 4, 4, 1, 2, 2, 2, 2, 0, 0, 1, 1, 3, 2, range(16), [1] * 4,
                           status=2))
    cases.append(conv_case("conv_filter_too_big", 1, 1, 3, 3, 1, 3, 3, 1, 1, 0, 0, 2, 2, 1, 1, [1] * 9, [1] * 9,
                           status=2))
    json.dump({"comment": __doc__.strip().splitlines()[0], "cases": cases}, open(OUT, "w"), indent=1)
    print(f"{len(cases)} cases -> {OUT}")


if __name__ == "__main__":
    main()
