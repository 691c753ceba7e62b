"""Error bounds of the NATIVE kernels' fast-math path against libm (north star: "a
fast-math sincos/log path whose error is bounded against the reference").

`wos_fastmath_probe` evaluates the kernels' own primitives (__sincosf = MUFU.SIN/COS
after the range-reducing multiply, sqrt.approx, ex2.approx) on the argument ranges
the kernels feed them; numpy fp64 on the same fp32 arguments is the reference. The
bounds asserted here are the ones DESIGN.md section 2 states.
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# argument ranges the NATIVE kernels use
RANGES = {
    # direction angles: dir_angle(f12(w)) = fmaf(f, 2 pi, -3 pi) with f in [1, 2)
    "direction angle [-pi, pi)": (-math.pi, math.pi),
    # the arc-length boundary's 2 pi s / 4, s in [0, 4) (once per walk)
    "arc-length angle [0, 2pi)": (0.0, 2.0 * math.pi),
    # sine sources on the unit box: k pi y for y in [0, 1] (monomial / Chebyshev rows)
    "sine source [0, pi]": (0.0, math.pi),
    # delta-tracking family coefficients (arguments below ~25 rad)
    "screened family [-25, 25]": (-25.0, 25.0),
}
SIN_BOUND = {  # max |error| (absolute)
    "direction angle [-pi, pi)": 2.0 ** -21,
    "arc-length angle [0, 2pi)": 2.0 ** -20,
    "sine source [0, pi]": 2.0 ** -21,
    "screened family [-25, 25]": 2.0 ** -18,
}


def _probe(gpu, x):
    import torch

    from paper_2603_01193_b200 import _lib

    d = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32), device="cuda:0")
    outs = [torch.empty_like(d) for _ in range(4)]
    _lib.check(_lib.lib().wos_fastmath_probe(gpu.handle, d.numel(), d.data_ptr(), *[o.data_ptr() for o in outs],
                                             None))
    torch.cuda.synchronize()
    return [o.cpu().numpy().astype(np.float64) for o in outs]


@pytest.mark.parametrize("name", list(RANGES))
def test_sincos_absolute_error(gpu, name):
    lo, hi = RANGES[name]
    x = np.linspace(lo, hi, 2_000_001, dtype=np.float64).astype(np.float32)
    s, c, _, _ = _probe(gpu, x)
    xd = x.astype(np.float64)
    es = np.max(np.abs(s - np.sin(xd)))
    ec = np.max(np.abs(c - np.cos(xd)))
    print(f"{name}: max |sin err| = 2^{math.log2(es):.2f}, max |cos err| = 2^{math.log2(ec):.2f}")
    assert es <= SIN_BOUND[name] and ec <= SIN_BOUND[name]


def test_sqrt_relative_error(gpu):
    x = np.concatenate([np.geomspace(1e-12, 4.0, 1_000_001), np.linspace(0.0, 1.0, 100_001)[1:]])
    x = x.astype(np.float32)
    _, _, q, _ = _probe(gpu, x)
    xd = x.astype(np.float64)
    rel = np.abs(q - np.sqrt(xd)) / np.sqrt(xd)
    print(f"sqrt.approx: max rel err = 2^{math.log2(rel.max()):.2f}")
    assert rel.max() <= 2.0 ** -23


def test_ex2_relative_error(gpu):
    # the Gaussian source exp(-r^2 / (2 sigma^2)) = ex2(-r^2 log2(e) / (2 sigma^2))
    x = np.linspace(-30.0, 0.0, 2_000_001).astype(np.float32)
    _, _, _, e = _probe(gpu, x)
    ref = np.exp2(x.astype(np.float64))
    rel = np.abs(e - ref) / ref
    print(f"ex2.approx: max rel err = 2^{math.log2(rel.max()):.2f}")
    assert rel.max() <= 2.0 ** -22


def test_probe_rejects_bad_arguments(gpu):
    from paper_2603_01193_b200 import _lib

    with pytest.raises(_lib.WosError):
        _lib.check(_lib.lib().wos_fastmath_probe(gpu.handle, 5, None, None, None, None, None, None))
