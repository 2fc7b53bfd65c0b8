"""jg_gemm (bf16, tcgen05) vs torch.matmul (cuBLAS) on every distinct GEMM shape of the 1-GPU
C4 training step (model.py forward / backward), interleaved (jg, cuBLAS, jg, cuBLAS, ...) so
both see the same clock / power state; best-of-rounds per side, SM clock sampled per case.

    python tools/bench_gemm.py [--json out.json]

Majors: 0 = K-major (row-major [m, k] / [n, k]), 1 = MN-major ([k, m] / [k, n]).
"""
import argparse
import json
import subprocess
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_05753_b200 import tensor as T  # noqa: E402

Tn, E, F, DT, DC = 16380, 4320, 4480, 8640, 4320
CASES = [  # name (where it runs per block / per step), m, n, k, a_major, b_major
    ("enc fwd NT", Tn, E, F, 0, 0),
    ("tok1 fwd TN | tok2 dX", E, DT, Tn, 1, 1),
    ("tok2 fwd NT | tok1 dX", Tn, E, DT, 0, 0),
    ("ch1/ch2 fwd NT", Tn, DC, E, 0, 0),
    ("dec fwd NT", Tn, F, E, 0, 0),
    ("dec dX NN", Tn, E, F, 0, 1),
    ("dec dW TN", F, E, Tn, 1, 1),
    ("ch1/ch2 dX NN", Tn, E, DC, 0, 1),
    ("ch1/ch2 dW TN", DC, E, Tn, 1, 1),
    ("tok1/tok2 dW NN", Tn, DT, E, 0, 1),
    ("enc dW TN", E, F, Tn, 1, 1),
]


def sm_clock():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                              "-i", "0"], capture_output=True, text=True, timeout=10).stdout.strip()
        c, p = out.split(",")
        return float(c), float(p)
    except Exception:  # noqa: BLE001
        return None, None


def timeit(fn, it=10):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--rounds", type=int, default=4)
    a = ap.parse_args()
    rows = []
    for name, m, n, k, am, bm in CASES:
        g = torch.Generator(device="cuda").manual_seed(0)
        A = torch.randn((m, k) if am == 0 else (k, m), device="cuda", generator=g).bfloat16()
        B = torch.randn((n, k) if bm == 0 else (k, n), device="cuda", generator=g).bfloat16()
        out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        At = A if am == 0 else A.t()
        Bt = B.t() if bm == 0 else B
        jg = lambda: T.gemm_into(out, A, B, am, bm, m, n, k)  # noqa: E731
        cb = lambda: torch.matmul(At, Bt)  # noqa: E731
        for _ in range(3):
            jg(), cb()
        torch.cuda.synchronize()
        t_jg, t_cb, clocks = [], [], []
        for _ in range(a.rounds):
            t_jg.append(timeit(jg))
            t_cb.append(timeit(cb))
            clocks.append(sm_clock()[0])
        ref = torch.matmul(At.float(), Bt.float())
        err = ((out.float() - ref).abs().max() / ref.abs().max()).item()
        fl = 2.0 * m * n * k
        r = {"case": name, "m": m, "n": n, "k": k, "a_major": am, "b_major": bm,
             "jg_ms": min(t_jg), "cublas_ms": min(t_cb), "jg_tflops": fl / min(t_jg) / 1e9,
             "cublas_tflops": fl / min(t_cb) / 1e9, "jg_over_cublas": min(t_cb) / min(t_jg), "rel_err": err,
             "sm_mhz": [c for c in clocks if c is not None]}
        rows.append(r)
        print(f"{name:24s} {m}x{n}x{k} ({am}{bm}): jg {r['jg_ms']:.3f} ms {r['jg_tflops']:.0f} TF/s | cuBLAS "
              f"{r['cublas_ms']:.3f} ms {r['cublas_tflops']:.0f} TF/s | jg/cuBLAS speed {r['jg_over_cublas']:.3f} | "
              f"err {err:.1e} | SM MHz {r['sm_mhz']}", flush=True)
        del A, B, out, ref
        torch.cuda.empty_cache()
    if a.json:
        json.dump({"device": torch.cuda.get_device_name(0), "rows": rows}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
