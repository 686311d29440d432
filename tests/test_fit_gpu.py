"""Device PerfModel::fit (include/slos_fit.h) against the reference's own
PerfModel::fit (perf_model.cpp:132-201) compiled in oracle/_ref: coefficients
bit-identical, same errors. The profile sets follow the reference's tests
(test_perf_model.cpp:90-113: clean and 2%-noise two-regime data, starved and flat
inputs; acceptance_main.cpp:629-648: the +-2% grid) plus random max-of-affine
models with 1-4 terms."""
import numpy as np
import pytest

from paper_2504_08784_b200 import fit as FT

pytestmark = pytest.mark.gpu


def _truth(terms, n, s):
    return np.max([k1 * n + k2 * s + b for k1, k2, b in terms], axis=0)


def _synth(terms, count, noise, seed):
    rng = np.random.default_rng(seed)
    n = rng.integers(1, 8193, count)
    s = rng.choice([0, 1, 2, 4, 8], count)
    lat = _truth(terms, n.astype(np.float64), s.astype(np.float64))
    if noise:
        lat = lat * (1.0 + rng.uniform(-noise, noise, count))
    return FT.as_samples(n, s, lat)


def _cases():
    desk = [(2.5e-5, 2e-3, 0.006), (0.0, 0.0, 0.02)]
    cases = [(_synth(desk, 8192, 0.0, 1), 2), (_synth(desk, 8192, 0.02, 2), 2)]
    rng = np.random.default_rng(3131)  # the acceptance grid: n = 8..8192 step 64, s in {0,2,5,8}
    n, s = np.meshgrid(np.arange(8, 8193, 64), [0, 2, 5, 8], indexing="ij")
    n, s = n.ravel(), s.ravel()
    lat = _truth([(2.5e-6, 2e-4, 0.003), (0.0, 0.0, 0.008)], n.astype(float), s.astype(float))
    cases.append((FT.as_samples(n, s, lat * (1.0 + rng.uniform(-0.02, 0.02, len(n)))), 2))
    for seed in range(24):  # random models, 1-4 terms, some with duplicate num_tokens
        r = np.random.default_rng(100 + seed)
        T = int(r.integers(1, 5))
        terms = [(float(r.uniform(0, 5e-5)), float(r.uniform(0, 3e-3)), float(r.uniform(0, 0.03))) for _ in range(T)]
        cnt = int(r.integers(3 * T, 3000))
        smp = _synth(terms, cnt, float(r.choice([0.0, 0.01, 0.05])), 1000 + seed)
        if seed % 3 == 0:
            smp["num_tokens"] = (smp["num_tokens"] // 256 + 1) * 256
        cases.append((smp, T if seed % 4 else max(1, T - 1)))
    return cases


def test_fit_matches_reference_bits():
    cases = _cases()
    by_T = {}
    for k, (smp, T) in enumerate(cases):
        by_T.setdefault(T, []).append(k)
    for T, ks in by_T.items():
        got, st = FT.fit_batch([cases[k][0] for k in ks], T)
        for j, k in enumerate(ks):
            want, wst = FT.reference_fit(cases[k][0], T)
            assert st[j] == wst == 0, (k, FT.ERR_SLUGS.get(int(st[j])), FT.ERR_SLUGS.get(wst))
            assert got[j].tobytes() == want.tobytes(), f"case {k} (T={T}): {got[j]} vs {want}"


def test_fit_errors_match_reference():
    desk = [(1e-4, 0.0, 0.01)]
    few = _synth(desk, 200, 0.0, 3)[:4]
    flat = FT.as_samples([100] * 12, [0] * 12, [0.02] * 12)
    got, st = FT.fit_batch([few, flat], 2)
    assert [FT.ERR_SLUGS[int(x)] for x in st] == ["insufficient-samples", "degenerate-samples"]
    assert FT.reference_fit(few, 2)[1] == st[0] and FT.reference_fit(flat, 2)[1] == st[1]
