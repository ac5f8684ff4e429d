"""Kernel-level timing of the step entry points (tsqr_proj / tsqr_update / tsqr_trmm / tsqr_gram)
at BASELINE cfg3 shapes (m = 2^22 rows), CUDA events on the current stream, median of reps.
Reports FP64 TFLOP/s (algorithmic flops) and HBM GB/s (algorithmic bytes) per call."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_04237_b200 as t  # noqa: E402


REPS = int(os.environ.get("KB_REPS", 7))
ONLY = os.environ.get("KB_ONLY", "")


def timeit(fn, reps=None):
    reps = reps or REPS
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    m = int(os.environ.get("KB_M", 1 << 22))
    n = 512
    A = t.colmajor_empty(m, n)
    A.normal_()
    A /= m ** 0.5
    out = {}
    Y = t.colmajor_empty(64, 448); Y.normal_()
    C = t.colmajor_empty(448, 64); C.normal_()
    Z = torch.triu(torch.randn(64, 64, dtype=torch.float64, device="cuda")).T.contiguous().T
    for (p, q) in ([] if ONLY and ONLY != "proj" else [(64, 448), (64, 192), (448, 64), (64, 64)]):
        ms = timeit(lambda: t.proj(A[:, :p], A[:, p:p + q]))
        fl, by = 2.0 * m * p * q, 8.0 * m * (p + q)
        out[f"proj_{p}x{q}"] = {"ms": ms, "tflops": fl / ms / 1e9, "gbs": by / ms / 1e6}
    for (p, q) in ([] if ONLY and ONLY != "update" else [(64, 448), (64, 256), (64, 128), (64, 64), (128, 64), (256, 64), (448, 64)]):
        S = (Y[:, :q] if p == 64 else C[:p, :q])
        ms = timeit(lambda: t.update(A[:, p:p + q], A[:, :p], S))
        fl, by = 2.0 * m * p * q, 8.0 * m * (p + 2 * q)
        out[f"update_{p}x{q}"] = {"ms": ms, "tflops": fl / ms / 1e9, "gbs": by / ms / 1e6}
    if ONLY and ONLY not in ("trmm", "misc"):
        return finish(out)
    ms = timeit(lambda: t.trmm(A[:, :64], Z))
    out["trmm_64"] = {"ms": ms, "tflops": m * 64 * 64 / ms / 1e9, "gbs": 16.0 * m * 64 / ms / 1e6}
    for bb in (128, 256):
        Zb = torch.triu(torch.randn(bb, bb, dtype=torch.float64, device="cuda")).T.contiguous().T
        ms = timeit(lambda: t.trmm(A[:, :bb], Zb))
        out[f"trmm_{bb}"] = {"ms": ms, "tflops": m * bb * bb / ms / 1e9, "gbs": 16.0 * m * bb / ms / 1e6}
        Wb = t.gram(A[:, :bb])
        ms = timeit(lambda: t.chol_inv(Wb))
        out[f"chol_inv_{bb}"] = {"ms": ms, "tflops": 0.0, "gbs": 0.0}
        ms = timeit(lambda: t.gram(A[:, :bb]))
        out[f"gram_{bb}"] = {"ms": ms, "tflops": m * bb * bb / ms / 1e9, "gbs": 8.0 * m * bb / ms / 1e6}
    W = t.gram(A[:, :64])
    ms = timeit(lambda: t.chol_inv(W))
    out["chol_inv_64"] = {"ms": ms, "tflops": 0.0, "gbs": 0.0}
    ms = timeit(lambda: t.gram(A[:, :64]))
    out["gram_64"] = {"ms": ms, "tflops": m * 64 * 64 / ms / 1e9, "gbs": 8.0 * m * 64 / ms / 1e6}
    finish(out)


def finish(out):
    for k, v in out.items():
        print(f"{k:16s} {v['ms']:8.3f} ms  {v['tflops']:7.2f} TF  {v['gbs']:8.0f} GB/s")
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "kbench.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
