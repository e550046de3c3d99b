"""Micro-benchmark of the tcgen05 GEMM on the Qwen3-8B linear shapes (T=4096)
against torch.matmul (cuBLAS) on the same box. CUDA-event timed, warmed up,
inputs > L2 rotated between iterations. Prints one JSON line per shape."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_27085_b200 import kernels  # noqa: E402

T = 4096
SHAPES = {  # name: (M, N, K, a_mn, b_mn, out_f32/acc)
    "qkv_fwd": (T, 6144, 4096, 0, 0, 0),
    "o_fwd": (T, 4096, 4096, 0, 0, 0),
    "gu_fwd": (T, 24576, 4096, 0, 0, 0),
    "down_fwd": (T, 4096, 12288, 0, 0, 0),
    "gu_dgrad": (T, 4096, 24576, 0, 1, 0),
    "gu_wgrad": (24576, 4096, T, 1, 1, 1),
    "down_wgrad": (4096, 12288, T, 1, 1, 1),
    "head_fwd_chunk": (1024, 151936, 4096, 0, 0, 0),
    "down_dgrad": (T, 12288, 4096, 0, 1, 0),
    # LoRA r=32 adapter GEMMs (gate/up linear: in 4096, out 24576)
    "lora_u": (T, 32, 4096, 0, 0, 0),          # U = X A^T
    "lora_du": (T, 32, 24576, 0, 1, 0),        # dU = dY B
    "lora_db": (24576, 32, T, 1, 1, 1),        # dB += dY^T U
    "lora_da": (32, 4096, T, 1, 1, 1),         # dA += dU^T X
    "lora_upd": (T, 24576, 32, 0, 0, 0),       # Y += U B^T (rank-r update)
}


def swiglu_case():
    """down dgrad + SwiGLU backward: fused epilogue vs GEMM then rp_swiglu_bwd"""
    m, h = 12288, 4096
    dy = torch.randn(T, h, device="cuda").to(torch.bfloat16)
    Wd = torch.randn(h, m, device="cuda").to(torch.bfloat16)
    gu = torch.randn(T, 2 * m, device="cuda").to(torch.bfloat16)
    dgu = torch.empty_like(gu)
    dact = torch.empty(T, m, device="cuda", dtype=torch.bfloat16)
    fused = bench(lambda: kernels.gemm_swiglu_bwd(dy, Wd, gu, dgu))
    gemm_only = bench(lambda: kernels.gemm(dy, Wd, dact, b_mn_major=True))
    two = bench(lambda: (kernels.gemm(dy, Wd, dact, b_mn_major=True),
                         kernels.swiglu_bwd(dact, gu, dgu)))
    X = torch.randn(T, h, device="cuda").to(torch.bfloat16)
    Wgu = torch.randn(2 * m, h, device="cuda").to(torch.bfloat16)
    act = torch.empty(T, m, device="cuda", dtype=torch.bfloat16)
    ffused = bench(lambda: kernels.gemm_swiglu_fwd(X, Wgu, gu, act))
    fgemm = bench(lambda: kernels.gemm(X, Wgu, gu))
    ftwo = bench(lambda: (kernels.gemm(X, Wgu, gu), kernels.swiglu_fwd(gu, act)))
    print(json.dumps({"gemm": "gu_fwd_swiglu", "fused_ms": round(ffused, 4),
                      "gemm_only_ms": round(fgemm, 4), "two_kernel_ms": round(ftwo, 4)}))
    print(json.dumps({"gemm": "down_dgrad_swiglu", "fused_ms": round(fused, 4),
                      "gemm_only_ms": round(gemm_only, 4), "two_kernel_ms": round(two, 4)}))


def bench(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    names = sys.argv[1:] or list(SHAPES)
    for name in names:
        if name == "swiglu":
            swiglu_case()
            continue
        M, N, K, a_mn, b_mn, f32 = SHAPES[name]
        A = torch.randn(*((K, M) if a_mn else (M, K)), device="cuda").to(torch.bfloat16)
        B = torch.randn(*((K, N) if b_mn else (N, K)), device="cuda").to(torch.bfloat16)
        D = torch.zeros(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
        ms = bench(lambda: kernels.gemm(A, B, D, a_mn_major=bool(a_mn), b_mn_major=bool(b_mn),
                                        accumulate=bool(f32)))
        Ar = A.t() if a_mn else A
        Br = B if b_mn else B.t()
        ms_ref = bench(lambda: torch.matmul(Ar, Br))
        tf = 2.0 * M * N * K / ms / 1e9
        print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "ms": round(ms, 4),
                          "tflops": round(tf, 1),
                          "cublas_ms": round(ms_ref, 4),
                          "cublas_tflops": round(2.0 * M * N * K / ms_ref / 1e9, 1)}))


if __name__ == "__main__":
    main()
