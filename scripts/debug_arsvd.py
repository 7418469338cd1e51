import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2512_16543_b200 import ops
from paper_2512_16543_b200.omega import normals_per_call_max
g = np.load('tests/golden/arsvd_cases.npz')
for (ci, eta, p, i_max) in [(6, 0.999, 5, 4), (0, 0.999, 5, 4), (3, 0.9, 5, 4)]:
    dA = g[f"c{ci}_dA"]; K = dA.shape[0]
    srng = np.random.default_rng([ci, int(eta * 1000), p, i_max])
    z = srng.standard_normal(normals_per_call_max(K, 2, p, i_max))
    dev = torch.device('cuda', 0)
    t = torch.from_numpy(dA).to(dev)[None].contiguous()
    om = torch.from_numpy(z).to(dev)[None].contiguous()
    cur = torch.zeros(1, dtype=torch.int64, device=dev)
    for im in (1, i_max):
        res = ops.arsvd(t, om, cur, eta, 2, p, im)
        torch.cuda.synchronize()
        D = res['D']
        ws = ops.workspace(dev, 0, 'arsvd')
        nel = 2 * D * K + D * D
        w = ws[:nel * 16].view(torch.complex128).cpu().numpy()
        Q = w[:D * K].reshape(D, K).T
        d = min(2 + p, K)
        print(ci, im, 'k', res['k_est'].item(), 'it', res['iters'].item(), 'S', res['S'][0, :4].cpu().numpy(),
              'QtQ err', np.abs(Q[:, :d].conj().T @ Q[:, :d] - np.eye(d)).max() if im == 1 else '')
        if im == 1:
            SQH = np.sqrt(0.5)
            Om = SQH * (z[:K * d].reshape(K, d) + 1j * z[K * d:2 * K * d].reshape(K, d))
            Y = dA @ Om
            Qr, R = np.linalg.qr(Y)
            print('   span err', np.linalg.norm(Q[:, :1] - Qr[:, :1] * (Qr[:, :1].conj().T @ Q[:, :1])))
            print('   sv ref', np.linalg.svd(Qr.conj().T @ dA, compute_uv=False)[:4])
            print('   sv of my Q', np.linalg.svd(Q[:, :d].conj().T @ dA, compute_uv=False)[:4])
