"""Stage split (CUDA events between stages) of one chunk of a BASELINE config.

    python scripts/stage_probe_cfg.py C3 [chunk] [dtype] [eta]
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2512_16543_b200 import scenario as S  # noqa: E402
from paper_2512_16543_b200.omega import DeviceOmegaStreams  # noqa: E402
from paper_2512_16543_b200.trajectory import TrajectoryConfig, TrajectoryRunner  # noqa: E402

name = sys.argv[1]
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 50
spec = S.CONFIGS[name]
if len(sys.argv) > 3:
    spec = spec.with_(dtype=sys.argv[3])
eta_wb = float(sys.argv[4]) if len(sys.argv) > 4 else spec.eta
dev = torch.device("cuda", 0)
trials = list(range(spec.B))
chans = S.DeviceChannels(spec, trials, dev)
tdt = torch.complex64 if spec.dtype == "c64" else torch.complex128
noise = torch.full((spec.B, spec.K), spec.noise_var, dtype=torch.float64, device=dev)
for eta in (eta_wb, None):
    cfg = TrajectoryConfig(alpha=spec.alpha, eta=eta, k_init=spec.k_init, p=spec.p,
                           i_max=spec.i_max)
    rn = TrajectoryRunner(spec.B, spec.K, spec.N, tdt, cfg, dev)
    st = None if eta is None else DeviceOmegaStreams.for_method(spec.seed, eta, trials, dev)
    for c in range(3):
        t0 = c * chunk
        H = chans.generate(t0, t0 + chunk)
        om = None if eta is None else st.window(chunk * rn.normals_per_step_max())
        rn.prof = [] if c == 2 else None
        r = rn.run_chunk(H, noise, om)
        if eta is not None:
            st.advance(r.consumed)
    torch.cuda.synchronize()
    tot = {}
    for nm, a, b in rn.prof:
        tot[nm] = tot.get(nm, 0.0) + a.elapsed_time(b)
    print(name, spec.dtype, "eta", eta, {k: round(v, 3) for k, v in tot.items()},
          "sum", round(sum(tot.values()), 3), "ms per", spec.B * chunk, "updates",
          "passes", r.spec_passes)
