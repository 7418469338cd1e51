import os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2512_16543_b200 import ops
cuda = torch.device('cuda', 0)
prof = len(sys.argv) > 1 and sys.argv[1] == "prof"
for K, N, B in [(64, 1024, 3), (128, 1024, 2), (256, 4096, 2), (48, 256, 2), (256, 256, 5)]:
    rng = np.random.default_rng(K + N)
    H = ((rng.standard_normal((B, K, N)) + 1j * rng.standard_normal((B, K, N))) * np.sqrt(0.5)).astype(np.complex64)
    alpha = K / 10.0
    H2 = H.astype(np.complex128)
    G = H2 @ np.conj(np.swapaxes(H2, 1, 2)) + alpha * np.eye(K)
    G = 0.5 * (G + np.conj(np.swapaxes(G, 1, 2)))
    Ainv = np.linalg.inv(G)
    noise = np.full((B, K), 0.1)
    Hd = torch.from_numpy(H).to(cuda)
    W = torch.empty(B, N, K, dtype=Hd.dtype, device=cuda)
    if prof: ops.prof_enable(True, cuda)
    pr = ops.precode_rate(Hd, torch.from_numpy(Ainv).to(cuda), 1.0, torch.from_numpy(noise).to(cuda), 1, W=W,
                          want_sinr=True, G_true=torch.from_numpy(G).to(cuda), alpha=alpha)
    torch.cuda.synchronize()
    if prof: print(ops.prof_collect(cuda)); ops.prof_enable(False, cuda)
    Wref = np.conj(np.swapaxes(H2, 1, 2)) @ Ainv
    s_ref = 1.0 / np.linalg.norm(Wref, axis=(1, 2))
    C = (H2 @ Wref) * s_ref[:, None, None]
    P = np.abs(C) ** 2
    sig = np.einsum("bii->bi", P)
    sinr = sig / (P.sum(2) - sig + noise)
    Wg = W.cpu().numpy()
    pr2 = ops.precode_rate(Hd.to(torch.complex128), torch.from_numpy(Ainv).to(cuda), 1.0, torch.from_numpy(noise).to(cuda), 1,
                          want_sinr=True, G_true=torch.from_numpy(G).to(cuda), alpha=alpha)
    print("   c128 rate", pr2["sum"].cpu().numpy() / np.log2(1 + sinr).sum(1) - 1)
    print(K, N, B, "W", max(np.linalg.norm(Wg[b]-Wref[b])/np.linalg.norm(Wref[b]) for b in range(B)),
          "rate", pr["sum"].cpu().numpy() / np.log2(1 + sinr).sum(1) - 1, "scale", pr["scale"].cpu().numpy()/s_ref - 1)
