"""GEMM micro-benchmark (dev tool, GPU box): TFLOP/s of the tcgen05 GEMM per orientation and
epilogue at the 22B layer's shapes, CUDA events over back-to-back launches.

    python tools/gemm_bench.py
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2205_05198_b200 as spl  # noqa: E402

EPI = {0: "store", 1: "bias", 2: "bias+gelu", 3: "x gelu'", 4: "fp32"}


def bench(M, N, K, a_mn, b_mn, epi, reps=20):
    A = torch.randn((K, M) if a_mn else (M, K), device="cuda").to(torch.bfloat16)
    B = torch.randn((K, N) if b_mn else (N, K), device="cuda").to(torch.bfloat16)
    bias = torch.randn(N, device="cuda")
    aux = torch.randn((M, N), device="cuda").to(torch.bfloat16)
    Cm = torch.empty((M, N), device="cuda", dtype=torch.float32 if epi == 4 else torch.bfloat16)
    C2 = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    be = C.c_int(-1)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def call():
        rc = spl.lib().spl_gemm_bf16(M, N, K, A.data_ptr(), A.shape[1], int(a_mn), B.data_ptr(),
                                     B.shape[1], int(b_mn), Cm.data_ptr(), N, epi,
                                     C.cast(bias.data_ptr(), C.POINTER(C.c_float)), C2.data_ptr(),
                                     aux.data_ptr(), N, st, C.byref(be))
        assert rc == 0, spl.lib().spl_last_error()

    for _ in range(3):
        call()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return 2.0 * M * N * K / (ms * 1e-3) / 1e12, ms


def layer_cases(h, tokens, t):
    """The 12 GEMMs of one layer rank at hidden h, s*b = tokens, tensor-parallel width t."""
    q, f = 3 * h // t, 4 * h // t
    return [("QKV fwd", tokens, q, h, 0, 1, 1), ("proj fwd", tokens, h, h // t, 0, 1, 0),
            ("FC1 fwd", tokens, f, h, 0, 1, 2), ("FC2 fwd", tokens, h, f, 0, 1, 0),
            ("FC2 dgrad", tokens, f, h, 0, 0, 3), ("FC1 dgrad", tokens, h, f, 0, 0, 0),
            ("proj dgrad", tokens, h // t, h, 0, 0, 0), ("QKV dgrad", tokens, h, q, 0, 0, 0),
            ("QKV wgrad", h, q, tokens, 1, 1, 4), ("proj wgrad", h // t, h, tokens, 1, 1, 4),
            ("FC1 wgrad", h, f, tokens, 1, 1, 4), ("FC2 wgrad", f, h, tokens, 1, 1, 4)]


SHAPES = {"22B": (6144, 8192), "175B": (12288, 2048), "530B": (20480, 2048), "1T": (25600, 2048)}


def main():
    if len(sys.argv) > 1:  # python tools/gemm_bench.py 175B [t]
        h, tokens = SHAPES[sys.argv[1]]
        t = int(sys.argv[2]) if len(sys.argv) > 2 else 1
        tot_f = tot_ms = 0.0
        for name, M, N, K, am, bm, epi in layer_cases(h, tokens, t):
            tf, ms = bench(M, N, K, am, bm, epi)
            tot_f += 2.0 * M * N * K
            tot_ms += ms
            print(f"{name:12s} M={M:6d} N={N:6d} K={K:6d} {EPI[epi]:10s} {ms:7.3f} ms {tf:7.0f} TFLOP/s",
                  flush=True)
        print(f"{sys.argv[1]} t={t}: {tot_ms:.3f} ms, {tot_f / tot_ms / 1e9:.0f} TFLOP/s overall")
        return
    cases = [  # name, M, N, K, a_mn, b_mn, epi
        ("QKV fwd", 8192, 18432, 6144, 0, 1, 1),
        ("FC1 fwd", 8192, 24576, 6144, 0, 1, 2),
        ("FC1 fwd (store)", 8192, 24576, 6144, 0, 1, 0),
        ("FC2 fwd", 8192, 6144, 24576, 0, 1, 0),
        ("FC2 dgrad", 8192, 24576, 6144, 0, 0, 3),
        ("FC2 dgrad (store)", 8192, 24576, 6144, 0, 0, 0),
        ("FC1 dgrad", 8192, 6144, 24576, 0, 0, 0),
        ("FC1 wgrad", 6144, 24576, 8192, 1, 1, 4),
        ("FC2 wgrad", 24576, 6144, 8192, 1, 1, 4),
        ("square K-major", 8192, 8192, 8192, 0, 0, 0),
        ("square fwd", 8192, 8192, 8192, 0, 1, 0),
        ("square wgrad", 8192, 8192, 8192, 1, 1, 4),
    ]
    for name, M, N, K, am, bm, epi in cases:
        tf, ms = bench(M, N, K, am, bm, epi)
        print(f"{name:20s} M={M:6d} N={N:6d} K={K:6d} A_MN={am} B_MN={bm} {EPI[epi]:10s} "
              f"{ms:7.3f} ms {tf:7.0f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
