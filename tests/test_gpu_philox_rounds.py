"""The NATIVE stream's generator on the GPU: round counts, layout, statistics.

* Philox4x32-R known answers: the GPU generator for R = 7 and R = 10 equals the
  exact-integer restatement (oracle.philox4x32_int) on random counters and keys;
  R = 10 equals Random123's published vectors (tests/test_gpu_replay.py).
* The opt-in 7-round stream (WalkConfig.philox_rounds = 7) walks exactly like the
  oracle's restatement with 7 rounds, differs from the 10-round stream, and its
  estimates agree with the reference form within combined standard errors.
* Statistics of the 7-round words in the walk's own counter layout (c0 = point id,
  c1 = 2 x block index, c2 = traj id): per-bit frequencies, serial correlation between a
  walk's consecutive blocks and between neighbouring walks, byte chi-square, and the
  strict avalanche criterion for single-bit counter changes. (Random123 reports
  Philox4x32-7 as the fewest rounds that pass TestU01 Crush; these tests check the
  properties the walk relies on in the layout it uses.)
* The Beta(2,2) radius fraction of the 3D source jump (a 12-bit index into the
  conditional-mean table, wos_walk.cuh jump3_source): over 1e9 draws of the production
  stream its index is uniform and its first two moments equal the table's (which
  differ from Beta(2,2)'s 1/2 and 3/10 by 0 and -1.0e-8).
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2603_01193_b200 import _lib, configs, estimate_arrays, walk_poisson_values
from paper_2603_01193_b200.walker import WalkConfig

pytestmark = pytest.mark.gpu


def _blocks(ctx, ctr_u32, k0, k1, rounds):
    """Philox4x32-R of [n, 4] uint32 counters (a CUDA int32 tensor) -> CUDA int32 [n, 4]."""
    out = torch.empty_like(ctr_u32)
    _lib.check(_lib.lib().wos_philox4x32_rounds(ctx.handle, ctr_u32.shape[0], ctr_u32.data_ptr(), k0, k1,
                                                rounds, out.data_ptr(), None))
    return out


@pytest.mark.parametrize("rounds", [7, 10, 1, 16])
def test_philox_rounds_known_answers(gpu, rounds):
    rng = np.random.default_rng(rounds)
    ctr = rng.integers(0, 2**32, size=(512, 4), dtype=np.uint64).astype(np.uint32)
    for k0, k1 in [(0, 0), (0xDEADBEEF, 7), (0xFFFFFFFF, 0xFFFFFFFF)]:
        got = _blocks(gpu, torch.from_numpy(ctr.view(np.int32)).cuda(), k0, k1, rounds)
        got = got.cpu().numpy().view(np.uint32)
        assert np.array_equal(got, O.philox4x32(ctr, k0, k1, rounds=rounds))
        for i in range(0, 512, 97):
            assert [int(v) for v in got[i]] == O.philox4x32_int(ctr[i], (k0, k1), rounds=rounds)


@pytest.mark.parametrize("cfg", [0, 4])
def test_seven_round_rows_match_oracle(gpu, cfg):
    w = configs.build(cfg)
    sel = np.arange(0, w.n_points, w.n_points // 48)[:48]
    T = 16
    pts = np.repeat(w.points[sel], T, axis=0)
    pid = np.repeat(w.point_ids[sel], T)
    tid = np.tile(np.arange(T), sel.size)
    sgn = np.ones(pts.shape[0])
    c7 = WalkConfig(eps_shell=w.cfg.eps_shell, max_steps=w.cfg.max_steps, rng_seed=w.cfg.rng_seed, philox_rounds=7)
    v7, s7, _ = walk_poisson_values(w.problems[0], pts, pid, tid, sgn, c7)
    v10, s10, _ = walk_poisson_values(w.problems[0], pts, pid, tid, sgn, w.cfg)
    vo, so, _ = O.walk_rows(w.problems[0], pts, pid, tid, sgn, seed=w.cfg.rng_seed, eps=w.cfg.eps_shell,
                            max_steps=w.cfg.max_steps, native=True, philox_rounds=7)
    assert np.mean(s7 == so) >= 0.99
    m = s7 == so
    rms = np.sqrt(np.mean(vo**2)) + 1e-30
    err = np.abs(v7[m] - vo[m]) / np.maximum(np.abs(vo[m]), rms)
    assert np.quantile(err, 0.99) < 1e-4
    assert np.mean(s7 == s10) < 0.5  # a different stream


@pytest.mark.parametrize("cfg,npts,L", [(0, 48, 4096), (4, 24, 4096)])
def test_seven_round_estimates_match_reference_form(gpu, cfg, npts, L):
    w = configs.build(cfg)
    idx = np.sort(np.random.default_rng(cfg).choice(w.n_points, size=npts, replace=False))
    w = w.subset(idx)
    c7 = WalkConfig(eps_shell=w.cfg.eps_shell, max_steps=w.cfg.max_steps, rng_seed=w.cfg.rng_seed, philox_rounds=7)
    mean, m2, n = estimate_arrays(w.problems, w.points, L, c7, point_ids=w.point_ids)
    om, om2, _ = O.estimate(w.problems, w.points, L, seed=w.cfg.rng_seed + 1, eps=w.cfg.eps_shell,
                            max_steps=w.cfg.max_steps, point_ids=w.point_ids)
    z = (mean - om) / np.sqrt(m2 / (n - 1) / n + om2 / (L - 1) / L + (1e-6 * np.maximum(1.0, np.abs(om)))**2)
    assert np.max(np.abs(z)) < 4.5
    assert 0.55 < float(np.sqrt(np.mean(z**2))) < 1.5


def _walk_counters(n_walks, n_steps, pid0=12345):
    """Counters of n_walks walks x n_steps blocks in the walk layout (c0 = point id,
    c1 = 2 x block index, c2 = traj id, c3 = 0), block-major within a walk."""
    s = torch.arange(n_steps, device="cuda", dtype=torch.int64)
    t = torch.arange(n_walks, device="cuda", dtype=torch.int64)
    c = torch.zeros((n_walks, n_steps, 4), dtype=torch.int64, device="cuda")
    c[:, :, 1] = 2 * s[None, :]
    c[:, :, 0] = pid0 + (t[:, None] // 256)
    c[:, :, 2] = t[:, None] % 256
    return c.reshape(-1, 4).to(torch.int32)


def _bits(words_i32):
    """[n, 4] int32 -> [n, 128] bool bits."""
    w = words_i32.to(torch.int64) & 0xFFFFFFFF
    sh = torch.arange(32, device=w.device, dtype=torch.int64)
    return ((w[:, :, None] >> sh) & 1).reshape(w.shape[0], 128)


def test_seven_round_stream_statistics(gpu):
    n_walks, n_steps = 1 << 14, 64  # 1M blocks = 128 Mbit
    w = _blocks(gpu, _walk_counters(n_walks, n_steps), 0x01234567, 0x89ABCDEF, 7)
    n = w.shape[0]
    # per-bit frequencies: each of 128 bits is fair within 5 sigma
    b = _bits(w).to(torch.float64)
    freq = b.mean(dim=0)
    assert torch.max(torch.abs(freq - 0.5)).item() < 5 * 0.5 / np.sqrt(n)
    # serial correlation of uniforms: a walk's consecutive blocks, and neighbouring walks
    u = (w.to(torch.int64) & 0xFFFFFFFF).to(torch.float64).reshape(n_walks, n_steps, 4) / 2**32 - 0.5
    lim = 5.0 / np.sqrt(n)
    for a, c in [(u[:, :-1], u[:, 1:]), (u[:-1], u[1:])]:
        for k in range(4):
            for j in range(4):
                r = (a[..., k] * c[..., j]).mean() / (1.0 / 12.0)
                assert abs(r.item()) < lim, (k, j, r.item())
    # words within a block are uncorrelated
    for k in range(4):
        for j in range(k + 1, 4):
            r = (u[..., k] * u[..., j]).mean() / (1.0 / 12.0)
            assert abs(r.item()) < lim
    # byte chi-square (255 dof): within a generous 6-sigma band
    by = torch.bincount(((w.to(torch.int64) & 0xFFFFFFFF)[:, :, None] >> torch.tensor([0, 8, 16, 24], device="cuda")
                         & 0xFF).reshape(-1), minlength=256).to(torch.float64)
    e = by.sum() / 256
    chi2 = (((by - e) ** 2) / e).sum().item()
    assert abs(chi2 - 255) < 6 * np.sqrt(2 * 255), chi2


@pytest.mark.parametrize("word,bit", [(0, 1), (0, 9), (0, 31), (2, 0), (2, 17), (1, 5), (3, 30)])
def test_seven_round_avalanche(gpu, word, bit):
    """Strict avalanche criterion: flipping one counter bit flips each of the 128 output
    bits with probability 1/2 (over 2^18 random counters, 6 sigma)."""
    n = 1 << 18
    g = torch.Generator(device="cuda").manual_seed(word * 64 + bit)
    c = torch.randint(-2**31, 2**31, (n, 4), device="cuda", dtype=torch.int64, generator=g).to(torch.int32)
    c2 = c.clone()
    c2[:, word] ^= int(np.array([1 << bit], dtype=np.uint32).view(np.int32)[0])
    a = _bits(_blocks(gpu, c, 7, 11, 7))
    b = _bits(_blocks(gpu, c2, 7, 11, 7))
    p = (a ^ b).to(torch.float64).mean(dim=0)
    assert torch.max(torch.abs(p - 0.5)).item() < 6 * 0.5 / np.sqrt(n)


@pytest.mark.parametrize("rounds", [10, 7])
def test_beta22_radius_moments_over_1e9_draws(gpu, rounds):
    """The radius fraction of the source jump (layout v4, wos_walk.cuh jump_source):
    index (wb >> 26) | (wa & 63) << 6 into the Beta(2,2) table, two jumps per
    block. Over 1.0e9 draws of the production stream the index is uniform, so E[t] and
    E[t^2] equal the table's exact means within 5 standard errors (and Beta(2,2)'s to
    ~1e-8)."""
    tab = torch.from_numpy(O.beta_table().astype(np.float64)).cuda()
    m1_exact, m2_exact = float(tab.mean()), float((tab * tab).mean())
    hist = torch.zeros(4096, dtype=torch.int64, device="cuda")
    total = 0
    chunk = 1 << 25
    n_chunks = 15  # 15 x 2^25 blocks x 2 jumps = 1.007e9 draws
    for k in range(n_chunks):
        i = torch.arange(chunk, device="cuda", dtype=torch.int64) + k * chunk
        c = torch.stack([77 + i // (1000 * 4096), 2 * (i % 1000), (i // 1000) % 4096, torch.zeros_like(i)],
                        dim=1).to(torch.int32)
        w = _blocks(gpu, c, 0x5EED, 0xC0FFEE, rounds).to(torch.int64) & 0xFFFFFFFF
        for wa, wb in ((w[:, 0], w[:, 1]), (w[:, 2], w[:, 3])):
            idx = (wb >> 26) | ((wa & 0x3F) << 6)
            hist += torch.bincount(idx, minlength=4096)
            total += chunk
    p = hist.to(torch.float64) / total
    e1 = (p * tab).sum().item()
    e2 = (p * tab * tab).sum().item()
    sd1 = np.sqrt(0.05 / total)        # Var[t] = 1/20
    sd2 = np.sqrt((1 / 7 - 0.09) / total)  # Var[t^2] = E[t^4] - E[t^2]^2 = 1/7 - 9/100
    assert abs(e1 - m1_exact) < 5 * sd1, (e1, m1_exact)
    assert abs(e2 - m2_exact) < 5 * sd2, (e2, m2_exact)
    # the 12-bit index itself is uniform (chi-square, 4095 dof, 6 sigma)
    e = total / 4096
    chi2 = (((hist.to(torch.float64) - e) ** 2) / e).sum().item()
    assert abs(chi2 - 4095) < 6 * np.sqrt(2 * 4095), chi2
