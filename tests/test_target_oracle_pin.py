"""Analytic-target harness (BASELINE.json configs[1]): pin the CPU restatement
(oracle_mix_run) to the reference composition (ref_mix_run: the UNMODIFIED
reference's KernelController, mh_accept, normal_quantile, RandomSequence and
Grid2D driven in lockstep) and to the committed fixtures under
tests/golden/target/ (tests/golden/make_golden_target.py).  CPU only.

Bar: bit-exact -- decision logs, final states, log densities, lambdas, update
counts, tallies and traces compare with ==.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

TARGET_DIR = os.path.join(GOLDEN, "target")
TARGET_CASES = sorted(f[:-4] for f in os.listdir(TARGET_DIR) if f.endswith(".npz"))
KEYS = ["x", "log_pi", "log_a", "log_f", "lambda_", "n", "tally_accept", "tally_visits", "trace"]


def load_target_case(name):
    from paper_2402_08273_b200.mix import MixTarget
    g = np.load(os.path.join(TARGET_DIR, name + ".npz"))
    d = {k: g[k] for k in g.files}
    d["config"] = json.loads(str(d["config"]))
    d["target"] = MixTarget(d["weights"], d["means"], d["covariances"])
    return d


@pytest.fixture(scope="module")
def oracle_built(oracle_lib):
    return oracle_lib


@pytest.mark.parametrize("name", TARGET_CASES)
def test_restatement_matches_reference_fixture(name, oracle_built):
    from oracle.abi import OracleMixConfig, mix_run
    g = load_target_case(name)
    o = mix_run(g["target"], OracleMixConfig(**g["config"]))
    for k in KEYS:
        assert np.array_equal(o[k], g[k]), k
    assert o["accepted"] == int(g["scalars"][0])
    assert o["acceptance_sum"] == g["scalars"][1]


@pytest.mark.parametrize("strategy,chains,seed", [("global", 1, 21), ("global", 5, 22), ("ra-grid", 7, 23),
                                                  ("fixed", 9, 24)])
def test_restatement_matches_reference_live(strategy, chains, seed, oracle_built):
    """Fresh seeds / targets: the restatement equals the reference composition."""
    from oracle.abi import REF_SO, OracleMixConfig, mix_run
    from paper_2402_08273_b200.mix import MixTarget
    if not os.path.exists(REF_SO):
        pytest.skip("reference harness not built")
    tgt = MixTarget.config2(seed, dim=6, n_comp=3)
    cfg = OracleMixConfig(strategy=strategy, grid_n=3, chains=chains, steps=600, seed=seed, log_steps=16,
                          lambda_init=-7.0 if strategy == "fixed" else 1.0)
    r = mix_run(tgt, cfg, reference=True)
    o = mix_run(tgt, cfg)
    for k in KEYS:
        assert np.array_equal(o[k], r[k]), k


def test_target_generator_matches_config2():
    """configs[1]: means in [0.2, 0.8]^8, eigenvalues in [1e-4, 1e-1], Dirichlet weights."""
    from paper_2402_08273_b200.mix import MixTarget
    t = MixTarget.config2(0)
    assert t.means.shape == (4, 8) and t.covariances.shape == (4, 8, 8)
    assert np.all((t.means >= 0.2) & (t.means <= 0.8))
    assert abs(t.weights.sum() - 1.0) < 1e-12 and np.all(t.weights > 0)
    for k in range(4):
        assert np.array_equal(t.covariances[k], t.covariances[k].T)
        ev = np.linalg.eigvalsh(t.covariances[k])
        assert ev.min() > 1e-4 * (1 - 1e-9) and ev.max() < 1e-1 * (1 + 1e-9)


def test_restatement_log_density_matches_numpy(oracle_built):
    """The oracle's whitened log density equals an independent numpy evaluation."""
    from oracle.abi import OracleMixConfig, mix_run
    from paper_2402_08273_b200.mix import MixTarget
    t = MixTarget.config2(4)
    o = mix_run(t, OracleMixConfig(strategy="global", chains=64, steps=300, seed=2))
    np.testing.assert_allclose(o["log_pi"], t.log_density(o["x"]), rtol=1e-10, atol=1e-9)


def test_pooled_equals_literal_for_one_chain(oracle_built):
    """With one chain the pooled rule batches exactly L visits, like the
    reference; alpha-hat differs only by the 2^-24 quantisation, which never
    crosses the target here (same lambda trajectory)."""
    from oracle.abi import OracleMixConfig, mix_run
    from paper_2402_08273_b200.mix import MixTarget
    t = MixTarget.config2(0)
    a = mix_run(t, OracleMixConfig(strategy="global", steps=2000, seed=3, adapt_mode="literal"))
    b = mix_run(t, OracleMixConfig(strategy="global", steps=2000, seed=3, adapt_mode="pooled"))
    assert np.array_equal(a["x"], b["x"])
    assert np.array_equal(a["trace"][:, [0, 1, 2, 3]], b["trace"][:, [0, 1, 2, 3]])
    np.testing.assert_allclose(a["trace"][:, 4], b["trace"][:, 4], atol=2 ** -24)


def test_error_contracts(oracle_built):
    from oracle.abi import OracleMixConfig, RenderError, mix_run
    from paper_2402_08273_b200.mix import MixTarget
    t = MixTarget.config2(0)
    bad = MixTarget(t.weights, t.means, t.covariances.copy())
    bad.covariances[1] = -bad.covariances[1]
    with pytest.raises(RenderError) as e:
        mix_run(bad, OracleMixConfig())
    assert e.value.code == 3 and "positive definite" in str(e.value)
    with pytest.raises(RenderError) as e:
        mix_run(t, OracleMixConfig(chains=0))
    assert e.value.code == 2


def test_autocorrelation_checker_matches_reference(ref_lib):
    """autocorrelation_time (core/diagnostics.cpp:87-127): the numpy checker
    equals the reference's function (AR(1) series with a known tau of
    (1 + phi) / (1 - phi)), including its error contract."""
    from oracle.abi import np_autocorrelation_time, ref_autocorrelation_time
    rng = np.random.default_rng(4)
    for phi in (0.0, 0.5, 0.9):
        e = rng.standard_normal(20000)
        x = np.empty_like(e)
        x[0] = e[0]
        for i in range(1, x.size):
            x[i] = phi * x[i - 1] + e[i]
        r = ref_autocorrelation_time(ref_lib, x)
        p = np_autocorrelation_time(x)
        np.testing.assert_allclose(p, r, rtol=1e-9)
        assert abs(r[0] - (1 + phi) / (1 - phi)) < 0.25 * (1 + phi) / (1 - phi) + 0.2
    assert ref_autocorrelation_time(ref_lib, np.ones(2000)) is None and np_autocorrelation_time(np.ones(2000)) is None
    assert ref_autocorrelation_time(ref_lib, np.arange(999.0)) is None and np_autocorrelation_time(np.arange(999.0)) is None
