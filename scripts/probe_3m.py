"""Probe: W = H^H A^-1 and the Gram at C5 c128 shapes (items = trials x steps of
one chunk), per-kernel CUDA-event times through lrz_prof (env LRZ_3M etc.)."""
import sys, os, torch
sys.path.insert(0, '.')
from paper_2512_16543_b200 import ops
dev = torch.device('cuda', 0)
K, N, items = int(os.environ.get('PK', 256)), int(os.environ.get('PN', 4096)), int(os.environ.get('PB', 640))
dt = torch.complex128 if os.environ.get('PDT', 'c128') == 'c128' else torch.complex64
torch.manual_seed(0)
H = torch.randn(items, K, N, dtype=dt, device=dev)
G = ops.gram(H, 25.6)
Ai = torch.linalg.inv(G[:4]).repeat(items // 4, 1, 1).contiguous()
noise = torch.full((items // 20, K), 0.1, dtype=torch.float64, device=dev)
W = torch.empty(items, N, K, dtype=dt, device=dev)
for rep in range(2):
    ops.prof_enable(True, dev)
    for _ in range(3):
        G = ops.gram(H, 25.6)
        pr = ops.precode_rate(H, Ai, 1.0, noise, 20, W=W, want_sinr=False, G_true=G, alpha=25.6)
    torch.cuda.synchronize()
    prof = ops.prof_collect(dev)
    ops.prof_enable(False, dev)
fl_w = 8.0 * K * K * N * items
fl_g = 4.0 * K * (K + 1) * N * items
for k, (ms, n) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
    extra = ''
    if k.startswith('w_dmma'):
        extra = ' %.1f TF/s (4-product flops)' % (fl_w / (ms / n) / 1e9)
    if k.startswith('gram_dmma_off'):
        extra = ' %.1f TF/s (4-product flops)' % (fl_g / (ms / n) / 1e9)
    print('%-28s %8.3f ms/launch x%d%s' % (k, ms / n, n, extra))
# accuracy against torch
ref = H[:2].conj().transpose(1, 2) @ Ai[:2]
print('W err', float((W[:2] - ref).norm() / ref.norm()))
Gr = H[:2] @ H[:2].conj().transpose(1, 2) + 25.6 * torch.eye(K, device=dev)
print('G err', float((G[:2] - Gr).norm() / Gr.norm()), 'herm', float((G[:2] - G[:2].conj().transpose(1, 2)).abs().max()))
