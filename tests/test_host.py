"""Host-side logic, the C ABI surface and the synthetic scenario (CPU only)."""

import math

import numpy as np
import pytest
import torch

from conftest import ROOT
from paper_2512_16543_b200 import _native, errors, lowrank, scenario as S
from paper_2512_16543_b200.omega import (consumed_by, normals_per_call_max, sketch_widths)
from paper_2512_16543_b200.trajectory import step_costs


def test_library_exports_every_header_symbol():
    from paper_2512_16543_b200 import build
    build.build()
    lib = _native.load()
    syms = _native.header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.lrz_version() == 1
    # workspace sizing is pure host arithmetic (CTA part + screening front end)
    base = 10 * (2 * 21 * 32 + 21 * 21) * 16
    assert lib.lrz_workspace_bytes(_native.WS_ARSVD, 1, 10, 32, 0, 21) >= base
    assert lib.lrz_workspace_bytes(_native.WS_RNG, 0, 4, 0, 100000, 0) > 4 * 100000 * 9


def test_sass_is_sm100a():
    """The built library carries sm_100a SASS (cuobjdump)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "--list-elf", str(_native.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(errors.NativeLibraryError):
        lowrank.gram_matrix(np.eye(3, dtype=complex), 1.0)


# -- reference cost-model tests (test_lowrank.py:286-319) -----------------------

def test_cost_reference_ratios():
    full = lowrank.cost_full(100)
    assert abs(lowrank.cost_wb_arsvd(100, 50) / full - 0.885) < 1e-12
    assert abs(lowrank.cost_wb_arsvd(100, 100) / full - 3.01) < 1e-12
    assert abs(lowrank.cost_wb_arsvd(100, 1) / full - 0.020101) < 1e-12


def test_cost_crossover_rank():
    full = lowrank.cost_full(100)
    ratios = np.array([lowrank.cost_wb_arsvd(100, r) / full for r in range(0, 101)])
    assert int(np.nonzero(ratios > 1.0)[0][0]) == 55


@pytest.mark.parametrize("K", [8, 16, 32, 64, 100, 128])
def test_cost_single_crossing(K):
    above = np.array([lowrank.cost_wb_arsvd(K, r) / lowrank.cost_full(K) > 1.0
                      for r in range(0, K + 1)])
    assert np.count_nonzero(above[1:] != above[:-1]) == 1 and above[-1]


def test_cost_monotone():
    for K in (2, 17, 256):
        for r in range(0, K):
            assert lowrank.cost_wb_arsvd(K, r + 1) > lowrank.cost_wb_arsvd(K, r)
    assert lowrank.sketch_cost(16, 3) == 16 * 16 * 3 + 9 * 16


def test_arsvd_config_validation():
    for kw in (dict(eta=0.0), dict(eta=1.5), dict(eta=0.5, k_init=0), dict(eta=0.5, p=-1),
               dict(eta=0.5, i_max=0)):
        with pytest.raises(ValueError):
            lowrank.ArSvdConfig(**kw)
    c = lowrank.ArSvdConfig(eta=1.0)
    assert (c.k_init, c.p, c.i_max) == (2, 1, 8)


def test_error_hierarchy_matches_reference():
    assert issubclass(errors.DimensionMismatchError, errors.SimulationError)
    assert issubclass(errors.SingularMatrixError, errors.SimulationError)
    assert issubclass(errors.SingularAuxiliaryError, errors.SimulationError)
    assert issubclass(errors.ZeroPrecoderError, errors.SimulationError)
    assert issubclass(errors.RangeError, errors.ConfigError)


def test_dimension_checks_before_device():
    with pytest.raises(errors.DimensionMismatchError):
        lowrank.direct_inverse(np.zeros((3, 4)))
    with pytest.raises(errors.DimensionMismatchError):
        lowrank.gram_delta(np.zeros((4, 8)), np.zeros((4, 9)))
    with pytest.raises(ValueError):
        lowrank.gram_matrix(np.eye(3, dtype=complex), -1.0)
    with pytest.raises(errors.DimensionMismatchError):
        lowrank.gram_matrix(np.zeros(3, dtype=complex), 1.0)
    st = lowrank.GramState(A=np.eye(2, dtype=complex), A_inv=np.eye(2, dtype=complex),
                           alpha=0.0, K=2)
    with pytest.raises(ValueError):
        lowrank.woodbury_update(st, lowrank.LowRankFactor.empty(2))


def test_sketch_schedule_and_consumption():
    assert sketch_widths(32, 2, 5, 4) == [7, 9, 13, 21]
    assert sketch_widths(16, 2, 5, 3) == [7, 9, 13]
    assert normals_per_call_max(32, 2, 5, 4) == 2 * 32 * (7 + 9 + 13 + 21)
    assert list(consumed_by([0, 1, 3, 4], 32, 2, 5, 4)) == [0, 448, 1856, 3200]
    # the C1 golden saw 928 and 224 (= 2*16*(7+9+13), 2*16*7)
    assert list(consumed_by([3, 1], 16, 2, 5, 3)) == [928, 224]


def test_step_costs():
    m = np.array([[0, 0, 1, 2]])
    k = np.array([[0, 20, 5, 0]])
    sk = np.array([[False, True, True, True]])
    c = step_costs(m, k, sk, 32)
    assert c[0, 0] == 32 ** 3
    assert c[0, 1] == 32 ** 3 + lowrank.sketch_cost(32, 20)
    assert c[0, 2] == lowrank.cost_wb_arsvd(32, 5)
    assert c[0, 3] == lowrank.cost_wb_arsvd(32, 0)


# -- synthetic scenario ------------------------------------------------

def test_configs_map_tolerance_and_cap():
    assert S.C1.i_max == 3 and S.C2.i_max == 4 and S.C5.i_max == 5
    assert math.isclose(S.C2.eta, 0.999)
    assert math.isclose(S.C2.alpha, 32 / 10.0) and math.isclose(S.C2.noise_var, 0.1)
    assert S.C3.N == 1024 and S.C5.N == 4096


def test_channel_shapes_power_and_determinism():
    spec = S.C1.with_(T=5)
    H1 = S.channels(spec)
    H2 = S.channels(spec)
    assert H1.shape == (1, 5, 16, 64) and H1.dtype == np.complex128
    assert np.array_equal(H1, H2)
    d = S.draw_trial(spec, 0)
    pw = np.mean(np.abs(H1[0]) ** 2, axis=(0, 2))
    # E|H_kn|^2 = beta_k (unit-modulus LOS + unit-variance scatter)
    assert np.allclose(pw / d.beta, 1.0, atol=0.35)
    assert S.channels(spec.with_(dtype="c64")).dtype == np.complex64
    # chunked generation equals one-shot
    a = S.trial_channels(spec, 0, 0, 5)
    b = np.concatenate([S.trial_channels(spec, 0, 0, 2), S.trial_channels(spec, 0, 2, 5)])
    assert np.array_equal(a, b)


def test_drift_is_small_per_step():
    spec = S.C2.with_(T=3, B=1)
    H = S.channels(spec)[0]
    rel = np.linalg.norm(H[1] - H[0]) / np.linalg.norm(H[0])
    assert 1e-4 < rel < 0.2


def test_exceptions_subclass_the_reference_classes_when_installed():
    """With the reference installed (baseline/_ref, or any `import leorzf`),
    a caller catching leorzf.errors.X catches this package's X
    (errors.py:28-50; cli.py:290-299).  Run in a fresh interpreter so the
    reference is importable before this package's errors module loads."""
    import os
    import subprocess
    import sys
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "leorzf").exists():
        pytest.skip("reference not installed in baseline/_ref")
    code = (
        "import leorzf.errors as E\n"
        "from paper_2512_16543_b200 import errors as X\n"
        "for n in ('ConfigError', 'SimulationError', 'DimensionMismatchError',\n"
        "          'SingularMatrixError', 'SingularAuxiliaryError', 'ZeroPrecoderError',\n"
        "          'EmptyInputError', 'BelowMinElevationError'):\n"
        "    assert issubclass(getattr(X, n), getattr(E, n)), n\n"
        "try:\n"
        "    raise X.SingularAuxiliaryError('x')\n"
        "except E.SimulationError:\n"
        "    print('ok')\n")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(ref), str(ROOT)]))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr


def test_device_log1p_restatement_matches_libm(tmp_path):
    """csrc/glibc_log1p.h (the device RNG's ziggurat-tail log1p) compiled for the
    host with gcc equals the libm log1p numpy's Generator calls, bit for bit, on
    the arguments the tail sees (-u, u in [0, 1)) and on every branch's range."""
    import ctypes
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    src = tmp_path / "l1p.c"
    src.write_text('#include "glibc_log1p.h"\n'
                   'void l1p(const double *x, double *y, long n)'
                   '{ for (long i = 0; i < n; ++i) y[i] = glibc_log1p(x[i]); }\n')
    so = tmp_path / "l1p.so"
    subprocess.run([gcc, "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-I",
                    str(ROOT / "paper_2512_16543_b200" / "csrc"), str(src), "-o", str(so), "-lm"],
                   check=True)
    twin = ctypes.CDLL(str(so))
    libm = ctypes.CDLL("libm.so.6")
    libm.log1p.restype = ctypes.c_double
    libm.log1p.argtypes = [ctypes.c_double]
    rng = np.random.default_rng(7)
    n = 400_000
    u = np.concatenate([
        rng.random(n),                                        # the tail's arguments
        rng.random(n) * 1e-6,                                 # k = 0, tiny |x|
        1.0 - rng.random(n) * 1e-3,                           # x -> -1
        np.ldexp(rng.random(n), -rng.integers(0, 60, n)),     # every exponent
        (1.0 + np.ldexp(rng.integers(0, 1 << 20, n).astype(np.float64), -52)) - 1.0,
        np.array([0.0, 2.0 ** -54, 2.0 ** -29, 0.2929, 0.5, 1.0 - 2.0 ** -53]),
    ])
    x = np.ascontiguousarray(-u)
    y = np.empty_like(x)
    twin.l1p(x.ctypes.data_as(ctypes.c_void_p), y.ctypes.data_as(ctypes.c_void_p),
             ctypes.c_long(x.size))
    # libm through ctypes, call by call (numpy's np.log1p ufunc may be a SIMD
    # variant, not the libm routine the Generator calls)
    want = np.array([libm.log1p(v) for v in x.tolist()])
    assert np.array_equal(y.view(np.uint64), want.view(np.uint64))
