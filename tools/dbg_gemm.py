import sys, torch
sys.path.insert(0, '.')
from paper_2604_27085_b200 import kernels
def mk(r, c, seed):
    g = torch.Generator(device='cuda').manual_seed(seed)
    return (torch.randn(r, c, device='cuda', generator=g) * 0.5).to(torch.bfloat16)
for (T, IN, OUT) in [(512, 384, 640), (512, 384, 512), (512, 256, 640), (64, 384, 640), (512, 512, 640)]:
    X, dY = mk(T, IN, 8), mk(T, OUT, 10)
    dW = torch.zeros(OUT, IN, device='cuda', dtype=torch.float32)
    kernels.gemm(dY, X, dW, a_mn_major=True, b_mn_major=True, accumulate=True)
    ref = dY.float().t() @ X.float()
    torch.cuda.synchronize()
    err = (dW - ref).abs()
    bad = (err > 1e-3 * ref.abs().max()).nonzero()
    print((T, IN, OUT), 'rel', ((dW - ref).norm() / ref.norm()).item(), 'nbad', len(bad))
    if len(bad):
        r, c = bad[:, 0], bad[:, 1]
        print('  rows', r.min().item(), r.max().item(), 'cols', c.min().item(), c.max().item())
        # which 32x32 chunks
        ch = set((int(a) // 32, int(b) // 32) for a, b in bad[:2000].tolist())
        print('  chunks', sorted(ch)[:20])
        print('  sample', dW[r[0], c[0]].item(), ref[r[0], c[0]].item())
