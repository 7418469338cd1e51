"""Per-kernel CUDA-event times (lrz_prof_*) of unpipelined WB chunks of a config.

    python scripts/kprof_cfg.py C5 c128 [chunk] [B] [nchunks]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2512_16543_b200 import ops, scenario as S  # noqa: E402
from paper_2512_16543_b200.omega import DeviceOmegaStreams  # noqa: E402
from paper_2512_16543_b200.trajectory import TrajectoryConfig, TrajectoryRunner  # noqa: E402

name, dt = sys.argv[1], sys.argv[2]
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 20
spec = S.CONFIGS[name].with_(dtype=dt)
if len(sys.argv) > 4:
    spec = spec.with_(B=int(sys.argv[4]))
nch = int(sys.argv[5]) if len(sys.argv) > 5 else 3
conv = len(sys.argv) > 6 and sys.argv[6] == "conv"
dev = torch.device("cuda", 0)
trials = list(range(spec.B))
chans = S.DeviceChannels(spec, trials, dev)
tdt = torch.complex64 if dt == "c64" else torch.complex128
noise = torch.full((spec.B, spec.K), spec.noise_var, dtype=torch.float64, device=dev)
cfg = TrajectoryConfig(alpha=spec.alpha, eta=None if conv else spec.eta, k_init=spec.k_init, p=spec.p,
                       i_max=spec.i_max)
rn = TrajectoryRunner(spec.B, spec.K, spec.N, tdt, cfg, dev)
st = DeviceOmegaStreams.for_method(spec.seed, spec.eta, trials, dev)
for c in range(nch):
    H = chans.generate(c * chunk, (c + 1) * chunk)
    om = None if conv else st.window(chunk * rn.normals_per_step_max())
    if c == 1:
        torch.cuda.synchronize()
        ops.prof_enable(True, dev)
        rn.prof = []
    r = rn.run_chunk(H, noise, om)
    if not conv:
        st.advance(r.consumed)
    del H
torch.cuda.synchronize()
k = ops.prof_collect(dev)
ops.prof_enable(False, dev)
n = nch - 1
print(f"{name} {dt} B={spec.B} chunk={chunk}: per chunk, ms")
stages = {}
for nm, a, b in rn.prof:
    stages[nm] = stages.get(nm, 0.0) + a.elapsed_time(b) / n
print("stages", {a: round(b, 2) for a, b in stages.items()}, "sum", round(sum(stages.values()), 1))
for nm, (ms, cnt) in sorted(k.items(), key=lambda kv: -kv[1][0]):
    print(f"  {nm:34s} {ms / n:9.3f} ms  {cnt / n:6.1f} launches")
