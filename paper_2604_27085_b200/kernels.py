"""Thin torch-tensor front-end to the sm_100a kernel C-ABI (include/rp/kernels.h).

Torch is only the allocator and stream provider here: every call goes
straight to libroundpipe_b200.so; there is no eager fallback. Used by the GPU
parity tests, smoke() and micro-benchmarks. The runtime (C++) calls the same
entry points directly.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _native

I32, I64, VP = C.c_int32, C.c_int64, C.c_void_p


class GemmArgs(C.Structure):
    _fields_ = [("M", I32), ("N", I32), ("K", I32),
                ("A", VP), ("lda", I64), ("a_mn_major", I32),
                ("B", VP), ("ldb", I64), ("b_mn_major", I32),
                ("D", VP), ("ldd", I64), ("out_f32", I32), ("accumulate", I32),
                ("R", VP), ("ldr", I64)]


def _lib():
    return _native.load()


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return VP(s.cuda_stream)


def _ptr(t):
    return VP(t.data_ptr()) if t is not None else VP(0)


def _check(code):
    return _native.check(_lib(), "rp_", code)


def gemm(A: torch.Tensor, B: torch.Tensor, D: torch.Tensor, *, a_mn_major=False,
         b_mn_major=False, accumulate=False, residual: torch.Tensor | None = None,
         stream=None):
    """D[M,N] (+)= op(A)[M,K] . op(B)[N,K]^T.

    A is [M,K] (a_mn_major=False) or [K,M] (True); B is [N,K] or [K,N].
    D bf16 (optionally + residual) or fp32 (optionally accumulated).
    """
    assert A.dtype == torch.bfloat16 and B.dtype == torch.bfloat16
    M = A.shape[1] if a_mn_major else A.shape[0]
    K = A.shape[0] if a_mn_major else A.shape[1]
    N = B.shape[1] if b_mn_major else B.shape[0]
    Kb = B.shape[0] if b_mn_major else B.shape[1]
    assert K == Kb and tuple(D.shape) == (M, N)
    assert D.dtype in (torch.bfloat16, torch.float32)
    for t in (A, B, D) + ((residual,) if residual is not None else ()):
        assert t.is_cuda and t.stride(1) == 1
    args = GemmArgs(M, N, K, _ptr(A), A.stride(0), int(a_mn_major),
                    _ptr(B), B.stride(0), int(b_mn_major),
                    _ptr(D), D.stride(0), int(D.dtype == torch.float32), int(accumulate),
                    _ptr(residual), residual.stride(0) if residual is not None else 0)
    f = _lib().rp_gemm_bf16
    f.restype = C.c_int
    rc = f(C.byref(args), _stream(stream))
    if rc:
        why = _lib().rp_gemm_last_error
        why.restype = C.c_char_p
        raise _native._ERRORS.get(rc, _native.NativeError)(
            rc, f"rp_gemm_bf16 M={M} N={N} K={K}: {why().decode()}")
    return D


def gemm_2seg(A, B, A2, B2, D, *, b_mn_major=False, residual=None, stream=None):
    """D = A[M,K] . op(B)^T + A2[M,K2] . op(B2)^T (+ residual): one GEMM with a second
    K segment (A, A2 K-major; B [N,K] / B2 [N,K2], or [K,N] / [K2,N] when b_mn_major)."""
    M, K = A.shape
    M2, K2 = A2.shape
    N = B.shape[1] if b_mn_major else B.shape[0]
    assert M2 == M and tuple(D.shape) == (M, N)
    args = GemmArgs(M, N, K, _ptr(A), A.stride(0), 0, _ptr(B), B.stride(0), int(b_mn_major),
                    _ptr(D), D.stride(0), int(D.dtype == torch.float32), 0,
                    _ptr(residual), residual.stride(0) if residual is not None else 0)
    f = _lib().rp_gemm_bf16_2seg
    f.restype = C.c_int
    _check(f(C.byref(args), _ptr(A2), I64(A2.stride(0)), _ptr(B2), I64(B2.stride(0)), I32(K2),
             _stream(stream)))
    return D


def gemm_swiglu_bwd(A: torch.Tensor, B: torch.Tensor, gu: torch.Tensor, dgu: torch.Tensor,
                    stream=None):
    """dgu = swiglu_bwd(dact = A[M,K] . B[K,N], gu) in one kernel (down-projection dgrad
    with the SwiGLU backward in its epilogue); gu, dgu are [M, 2N] bf16."""
    M, K = A.shape
    Kb, N = B.shape
    assert K == Kb and tuple(gu.shape) == (M, 2 * N) and tuple(dgu.shape) == (M, 2 * N)
    for t in (A, B, gu, dgu):
        assert t.is_cuda and t.stride(1) == 1 and t.dtype == torch.bfloat16
    args = GemmArgs(M, N, K, _ptr(A), A.stride(0), 0, _ptr(B), B.stride(0), 1,
                    _ptr(dgu), dgu.stride(0), 0, 0, _ptr(gu), gu.stride(0))
    f = _lib().rp_gemm_swiglu_bwd
    f.restype = C.c_int
    _check(f(C.byref(args), _stream(stream)))
    return dgu


def gemm_swiglu_fwd(A: torch.Tensor, W_gu: torch.Tensor, gu: torch.Tensor, act: torch.Tensor,
                    stream=None):
    """gu = A[M,K] . W_gu[2N,K]^T and act = silu(gu[:, :N]) * gu[:, N:] in one kernel."""
    M, K = A.shape
    N2, Kb = W_gu.shape
    N = N2 // 2
    assert K == Kb and N2 == 2 * N and tuple(gu.shape) == (M, N2) and tuple(act.shape) == (M, N)
    for t in (A, W_gu, gu, act):
        assert t.is_cuda and t.stride(1) == 1 and t.dtype == torch.bfloat16
    args = GemmArgs(M, N, K, _ptr(A), A.stride(0), 0, _ptr(W_gu), W_gu.stride(0), 0,
                    _ptr(gu), gu.stride(0), 0, 0, None, 0)
    f = _lib().rp_gemm_swiglu_fwd
    f.restype = C.c_int
    _check(f(C.byref(args), _ptr(act), I64(act.stride(0)), _stream(stream)))
    return act


class AdamHParams(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
                ("eps", C.c_float), ("weight_decay", C.c_float), ("grad_scale", C.c_float)]


def _call(name, *args):
    f = getattr(_lib(), name)
    f.restype = C.c_int
    return _check(f(*args))


F = C.c_float


def rmsnorm_fwd(x, w, y, rstd, eps=1e-6, stream=None):
    rows, h = x.shape
    _call("rp_rmsnorm_fwd", _ptr(x), I64(x.stride(0)), _ptr(w), _ptr(y), I64(y.stride(0)),
          _ptr(rstd), I32(rows), I32(h), F(eps), _stream(stream))


def rmsnorm_bwd(dy, x, w, rstd, dx32=None, dx16=None, dw=None, dres=None, stream=None):
    rows, h = x.shape
    _call("rp_rmsnorm_bwd", _ptr(dy), _ptr(x), _ptr(w), _ptr(rstd), _ptr(dres), _ptr(dx32),
          _ptr(dx16), _ptr(dw), I32(rows), I32(h), _stream(stream))


def qk_norm_rope_fwd(qkv, nq, nk, hd, qw, kw, cos_sin, seq, q_out, k_out, rstd_q, rstd_k,
                     eps=1e-6, stream=None):
    T = qkv.shape[0]
    _call("rp_qk_norm_rope_fwd", _ptr(qkv), I64(qkv.stride(0)), I32(nq), I32(nk), I32(hd),
          _ptr(qw), _ptr(kw), _ptr(cos_sin), I32(seq), _ptr(q_out), _ptr(k_out), _ptr(rstd_q),
          _ptr(rstd_k), I32(T), F(eps), _stream(stream))


def qk_norm_rope_bwd(dq, dk, qkv, nq, nk, hd, qw, kw, rstd_q, rstd_k, cos_sin, seq, dqkv,
                     dqw, dkw, stream=None):
    T = qkv.shape[0]
    _call("rp_qk_norm_rope_bwd", _ptr(dq), _ptr(dk), _ptr(qkv), I64(qkv.stride(0)), I32(nq),
          I32(nk), I32(hd), _ptr(qw), _ptr(kw), _ptr(rstd_q), _ptr(rstd_k), _ptr(cos_sin),
          I32(seq), _ptr(dqkv), I64(dqkv.stride(0)), _ptr(dqw), _ptr(dkw), I32(T),
          _stream(stream))


def swiglu_fwd(gu, act, stream=None):
    T, m = act.shape
    _call("rp_swiglu_fwd", _ptr(gu), _ptr(act), I64(T), I32(m), _stream(stream))


def swiglu_bwd(dact, gu, dgu, stream=None):
    T, m = dact.shape
    _call("rp_swiglu_bwd", _ptr(dact), _ptr(gu), _ptr(dgu), I64(T), I32(m), _stream(stream))


def embed_fwd(ids, table, out, stream=None):
    T, h = out.shape
    _call("rp_embed_fwd", _ptr(ids), _ptr(table), _ptr(out), I32(T), I32(h), _stream(stream))


def embed_bwd(ids, dx, dE, stream=None):
    T, h = dx.shape
    _call("rp_embed_bwd", _ptr(ids), _ptr(dx), _ptr(dE), I32(T), I32(h), _stream(stream))


def ce_fwd_bwd(logits, labels, grad_scale, loss_sum, row_lse=None, stream=None):
    rows, V = logits.shape
    _call("rp_ce_fwd_bwd", _ptr(logits), I64(logits.stride(0)), _ptr(labels), I32(rows), I32(V),
          F(grad_scale), _ptr(loss_sum), _ptr(row_lse), _stream(stream))


def adamw(master, m, v, grad, w16, step, lr=1e-4, beta1=0.9, beta2=0.95, eps=1e-8,
          weight_decay=0.0, grad_scale=1.0, stream=None):
    hp = AdamHParams(lr, beta1, beta2, eps, weight_decay, grad_scale)
    _call("rp_adamw", _ptr(master), _ptr(m), _ptr(v), _ptr(grad), _ptr(w16),
          I64(master.numel()), C.byref(hp), I32(step), _stream(stream))


def attn_fwd_tc(q, k, v, o, lse, seq, nq, nk, hd, scale=None, stream=None):
    T = q.shape[0]
    scale = scale if scale is not None else hd ** -0.5
    _call("rp_attn_fwd_tc", _ptr(q), I64(q.stride(0)), _ptr(k), I64(k.stride(0)), _ptr(v),
          I64(v.stride(0)), _ptr(o), I64(o.stride(0)), _ptr(lse), I32(T), I32(seq), I32(nq),
          I32(nk), I32(hd), F(scale), _stream(stream))


def attn_bwd_tc(q, k, v, o, do, lse, dq, dk, dv, delta, seq, nq, nk, hd, scale=None,
                stream=None, dkv_acc=None):
    T = q.shape[0]
    scale = scale if scale is not None else hd ** -0.5
    if dkv_acc is None:
        dkv_acc = torch.empty(2 * T * nk * hd, device=q.device, dtype=torch.float32)
    _call("rp_attn_bwd_tc", _ptr(q), I64(q.stride(0)), _ptr(k), I64(k.stride(0)), _ptr(v),
          I64(v.stride(0)), _ptr(o), I64(o.stride(0)), _ptr(do), I64(do.stride(0)), _ptr(lse),
          _ptr(dq), I64(dq.stride(0)), _ptr(dk), I64(dk.stride(0)), _ptr(dv), I64(dv.stride(0)),
          _ptr(delta), _ptr(dkv_acc), I32(T), I32(seq), I32(nq), I32(nk), I32(hd), F(scale),
          _stream(stream))


def rope_table(seq, hd, theta=1e6):
    """float2 (cos, sin) table [seq, hd/2], computed in float64 then rounded."""
    import numpy as np
    inv = 1.0 / (theta ** (np.arange(0, hd, 2, dtype=np.float64) / hd))
    ang = np.arange(seq, dtype=np.float64)[:, None] * inv[None, :]
    tab = np.stack([np.cos(ang), np.sin(ang)], axis=-1).astype(np.float32)
    return torch.from_numpy(np.ascontiguousarray(tab))


# ---- mixture of experts (include/rp/kernels.h, csrc/kernels/moe.cu) ------------------
def gemm_grouped(A, B, D, row_off, groups, b_group_rows, *, b_mn_major=False, gu=None,
                 stream=None):
    """Rows [row_off[e], row_off[e+1]) of A [M,K] / D [M,N] times expert e's block of B
    (K-major [groups*N, K] or MN-major [groups*K, N]). gu given: the SwiGLU-backward
    epilogue (D = dgu [M, 2N], B MN-major)."""
    M, K = A.shape
    N = B.shape[1] if b_mn_major else b_group_rows
    args = GemmArgs(M, N, K, _ptr(A), A.stride(0), 0, _ptr(B), B.stride(0), int(b_mn_major),
                    _ptr(D), D.stride(0), 0, 0, _ptr(gu), gu.stride(0) if gu is not None else 0)
    f = _lib().rp_gemm_grouped
    f.restype = C.c_int
    _check(f(C.byref(args), _ptr(row_off), I32(groups), I32(b_group_rows),
             I32(1 if gu is not None else 0), _stream(stream)))
    return D


def moe_route(logits, k, norm_topk, topk_idx, topk_w, counts, stream=None):
    T, E = logits.shape
    _call("rp_moe_route", _ptr(logits), I32(T), I32(E), I32(k), I32(int(norm_topk)),
          _ptr(topk_idx), _ptr(topk_w), _ptr(counts), _stream(stream))


def moe_permute(x, k, topk_idx, topk_w, counts, offsets, cursor, pos, w_s, xs, stream=None):
    T, h = x.shape
    E = counts.shape[0]
    _call("rp_moe_permute", _ptr(x), I64(x.stride(0)), I32(T), I32(h), I32(k), I32(E),
          _ptr(topk_idx), _ptr(topk_w), _ptr(counts), _ptr(offsets), _ptr(cursor), _ptr(pos),
          _ptr(w_s), _ptr(xs), _stream(stream))


def moe_gather(x, k, pos, xs, stream=None):
    T, h = x.shape
    _call("rp_moe_gather", _ptr(x), I64(x.stride(0)), I32(T), I32(h), I32(k), _ptr(pos),
          _ptr(xs), _stream(stream))


def moe_combine(ys, pos, topk_w, k, out, res=None, stream=None):
    T, h = out.shape
    _call("rp_moe_combine", _ptr(ys), _ptr(pos), _ptr(topk_w), I32(T), I32(k), I32(h),
          _ptr(res), I64(res.stride(0) if res is not None else 0), _ptr(out),
          I64(out.stride(0)), _stream(stream))


def moe_combine_bwd(dxs, pos, k, dh32, dh, stream=None):
    T, h = dh.shape
    _call("rp_moe_combine_bwd", _ptr(dxs), _ptr(pos), I32(T), I32(k), I32(h), _ptr(dh32),
          _ptr(dh), I64(dh.stride(0)), _stream(stream))


def moe_swiglu_bwd(dact, gu, w_s, dgu, dw_s, stream=None):
    rows, m = dact.shape
    _call("rp_moe_swiglu_bwd", _ptr(dact), _ptr(gu), _ptr(w_s), I64(rows), I32(m), _ptr(dgu),
          _ptr(dw_s), _stream(stream))


def moe_router_bwd(logits, k, norm_topk, topk_idx, pos, dw_s, dlogits, stream=None):
    T, E = logits.shape
    _call("rp_moe_router_bwd", _ptr(logits), I32(T), I32(E), I32(k), I32(int(norm_topk)),
          _ptr(topk_idx), _ptr(pos), _ptr(dw_s), _ptr(dlogits), _stream(stream))
