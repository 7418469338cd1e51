"""Pass time of a config with / without cross-chunk pipelining for several chunk sizes.

    python scripts/pipe_probe.py C2 c128 0.9 50,100,200
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2512_16543_b200 import scenario as S  # noqa: E402
from paper_2512_16543_b200.omega import DeviceOmegaStreams  # noqa: E402
from paper_2512_16543_b200.trajectory import TrajectoryConfig, TrajectoryRunner  # noqa: E402

name, dt, eta = sys.argv[1], sys.argv[2], float(sys.argv[3])
chunks = [int(x) for x in sys.argv[4].split(",")]
spec = S.CONFIGS[name].with_(dtype=dt)
dev = torch.device("cuda", 0)
trials = list(range(spec.B))
chans = S.DeviceChannels(spec, trials, dev)
H_all = chans.generate(0, spec.T)
tdt = torch.complex64 if dt == "c64" else torch.complex128
noise = torch.full((spec.B, spec.K), spec.noise_var, dtype=torch.float64, device=dev)
st = DeviceOmegaStreams.for_method(spec.seed, eta, trials, dev)
cur = torch.cuda.current_stream(dev)
back = torch.cuda.Stream(dev, priority=-1)
flags = torch.zeros(2, dtype=torch.int32, device=dev)


def one(ch, pipe):
    cfg = TrajectoryConfig(alpha=spec.alpha, eta=eta, k_init=spec.k_init, p=spec.p,
                           i_max=spec.i_max)
    rn = TrajectoryRunner(spec.B, spec.K, spec.N, tdt, cfg, dev)
    st.raw.zero_()
    st.consumed_total.zero_()
    evs = []
    Hs = [H_all[:, t0:t0 + ch].contiguous() for t0 in range(0, spec.T, ch)]
    for i, H in enumerate(Hs):
        if pipe and i >= 2:
            cur.wait_event(evs[i - 2])
        om = st.window(H.shape[1] * rn.normals_per_step_max())
        if pipe:
            r = rn.run_chunk(H, noise, om, sync=False, back_stream=back)
            flags.add_(r.flags)
            e = torch.cuda.Event()
            e.record(back)
            evs.append(e)
        else:
            r = rn.run_chunk(H, noise, om)
        st.advance(r.consumed)
    cur.wait_stream(back)


for ch in chunks:
    for pipe in (False, True):
        one(ch, pipe)
        torch.cuda.synchronize()
        flags.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            one(ch, pipe)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(name, dt, eta, "chunk", ch, "pipelined" if pipe else "sync", f"{ms:.2f} ms",
              f"{spec.B * spec.T / ms * 1e3:.0f} updates/s", "flags", flags.tolist())
