"""GPU parity of the analytic-target harness (BASELINE.json configs[1];
include/ramlt_mix.h) against the reference composition's fixtures
(tests/golden/target/, made by tests/golden/make_golden_target.py from the
UNMODIFIED reference's controller / accept / quantile / RNG) and against the
restatement oracle run live.

Bars:
  * f64 + PCG32 + literal rule: decision flags bit-exact, a within rtol 1e-9
    (libdevice vs glibc exp/log/erfc differ by ulps), lambda / n / tallies /
    trace equal (lambda moves in exact +-gamma steps, so equal trajectories
    give bit-equal lambdas), final states within 1e-9.
  * f64 + Philox (+ pooled rule): the same bar against the oracle's Philox build.
  * f32 production: statistical -- acceptance near the 0.5 target, lambda and
    the sample mean of the final states close to the f64 oracle's.
"""
import numpy as np
import pytest

from test_target_oracle_pin import TARGET_CASES, load_target_case

pytestmark = pytest.mark.gpu


def gpu_run(target, steps, log_steps=0, **kw):
    from paper_2402_08273_b200.mix import MixConfig, MixEngine
    kw.setdefault("trace_enabled", True)
    eng = MixEngine(target, MixConfig(log_steps=log_steps, **kw))
    eng.init_chains()
    eng.run(steps)
    x, lp = eng.state()
    lam, n, acc, vis = eng.regions()
    a, f = eng.decisions(log_steps) if log_steps else (None, None)
    out = dict(x=x, log_pi=lp, lambda_=lam, n=n, tally_accept=acc, tally_visits=vis, trace=eng.trace(),
               log_a=a, log_f=f, stats=eng.stats())
    eng.close()
    return out


def assert_same(g, o, tallies_rtol=1e-9):
    np.testing.assert_array_equal(o["log_f"], g["log_f"])
    np.testing.assert_allclose(o["log_a"], g["log_a"], rtol=1e-9, atol=1e-300)
    np.testing.assert_array_equal(o["lambda_"], g["lambda_"])
    np.testing.assert_array_equal(o["n"], g["n"])
    np.testing.assert_array_equal(o["tally_visits"], g["tally_visits"])
    np.testing.assert_allclose(o["tally_accept"], g["tally_accept"], rtol=tallies_rtol)
    assert o["trace"].shape == g["trace"].shape
    np.testing.assert_array_equal(o["trace"][:, :4], g["trace"][:, :4])
    np.testing.assert_allclose(o["trace"][:, 4], g["trace"][:, 4], rtol=1e-9)
    np.testing.assert_allclose(o["x"], g["x"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(o["log_pi"], g["log_pi"], rtol=1e-9)


@pytest.mark.parametrize("coop", [True, False])
@pytest.mark.parametrize("name", TARGET_CASES)
def test_f64_pcg_matches_reference(name, coop):
    """Persistent cooperative kernel and per-step launches, vs the reference."""
    g = load_target_case(name)
    c = g["config"]
    o = gpu_run(g["target"], c["steps"], log_steps=c["log_steps"], strategy=c["strategy"],
                grid_n=c["grid_n"], chains=c["chains"], seed=c["seed"], lambda_init=c["lambda_init"],
                precision="f64", rng="pcg32", adapt_mode="literal", cooperative=coop)
    assert_same(g, o)


@pytest.mark.parametrize("strategy,chains,mode", [("global", 300, "pooled"), ("ra-grid", 300, "pooled"),
                                                  ("global", 64, "literal"), ("ra-grid", 64, "literal"),
                                                  ("fixed", 500, "pooled")])
@pytest.mark.parametrize("coop", [True, False])
def test_f64_philox_matches_oracle(strategy, chains, mode, coop):
    """D = 8 / K = 4 with Philox takes the batched-draw step (mix_step_px8)."""
    from oracle.abi import OracleMixConfig, mix_run
    from paper_2402_08273_b200.mix import MixTarget
    t = MixTarget.config2(5)
    kw = dict(strategy=strategy, grid_n=4, chains=chains, seed=17, log_steps=24,
              lambda_init=-8.0 if strategy == "fixed" else 1.0)
    o = mix_run(t, OracleMixConfig(steps=300, rng="philox", adapt_mode=mode, **kw))
    gpu = gpu_run(t, 300, precision="f64", rng="philox", adapt_mode=mode, cooperative=coop, **kw)
    assert_same(o, gpu)


def test_f64_philox_sharded_fixed_large():
    """65,536 chains (the configs[1] count), Fixed: decisions of two chain
    windows equal the oracle run on those global chain ids alone."""
    from oracle.abi import OracleMixConfig, mix_run
    from paper_2402_08273_b200.mix import MixTarget
    t = MixTarget.config2(0)
    C = 65536
    gpu = gpu_run(t, 16, log_steps=16, strategy="fixed", chains=C, seed=5, lambda_init=-8.0,
                  precision="f64", rng="philox")
    for off in (0, C - 48):
        o = mix_run(t, OracleMixConfig(strategy="fixed", chains=48, chain_offset=off, chains_total=C, steps=16,
                                       seed=5, lambda_init=-8.0, rng="philox", log_steps=16))
        np.testing.assert_array_equal(gpu["log_f"][off:off + 48], o["log_f"])
        np.testing.assert_allclose(gpu["log_a"][off:off + 48], o["log_a"], rtol=1e-9, atol=1e-300)
        np.testing.assert_allclose(gpu["x"][off:off + 48], o["x"], atol=1e-9)


def test_external_exchange_equals_single_handle():
    """The sharded path (run one step, exchange, apply) on one handle gives
    the same chains and lambda trajectory as the fused cooperative kernel."""
    from paper_2402_08273_b200.mix import MixConfig, MixEngine, MixTarget
    t = MixTarget.config2(1)
    kw = dict(strategy="ra-grid", grid_n=4, chains=2000, seed=3, precision="f64", rng="philox",
              adapt_mode="pooled", trace_enabled=True)
    a = gpu_run(t, 120, **kw)
    eng = MixEngine(t, MixConfig(**kw))
    eng.init_chains()
    eng.set_external_adaptation(True)
    for _ in range(120):
        eng.run(1)
        eng.adapt_apply()
    x, _ = eng.state()
    lam, n, _, _ = eng.regions()
    tr = eng.trace()
    eng.close()
    np.testing.assert_array_equal(x, a["x"])
    np.testing.assert_array_equal(lam, a["lambda_"])
    np.testing.assert_array_equal(n, a["n"])
    np.testing.assert_array_equal(tr, a["trace"])


def test_f32_config2_statistics():
    """configs[1] at full chain count (65,536 chains), fp32 production build,
    1,024 steps: acceptance targets 0.5, lambda agrees with the f64 oracle, and
    the pooled final-state mean matches the oracle's (4,096-chain run) within
    5 standard errors per coordinate."""
    from oracle.abi import OracleMixConfig, mix_run
    from paper_2402_08273_b200.mix import MixTarget
    t = MixTarget.config2(0)
    steps = 1024
    g = gpu_run(t, steps, strategy="global", chains=65536, seed=1, precision="f32", rng="philox")
    o = mix_run(t, OracleMixConfig(strategy="global", chains=4096, steps=steps, seed=1, rng="philox",
                                   adapt_mode="pooled"))
    s = g["stats"]
    assert s.proposals == 65536 * steps
    assert abs(s.mean_acceptance - o["mean_acceptance"]) < 0.02, (s.mean_acceptance, o["mean_acceptance"])
    assert abs(g["lambda_"][0] - o["lambda_"][0]) < 0.3, (g["lambda_"], o["lambda_"])
    mg, mo = g["x"].mean(0), o["x"].mean(0)
    se = np.sqrt(o["x"].var(0) / 4096 + g["x"].var(0) / 65536)
    assert np.all(np.abs(mg - mo) < 5 * se + 1e-6), (mg, mo, se)
    # late acceptance near the target (the controller converged)
    late = g["trace"][-100:, 4]
    assert abs(late.mean() - 0.5) < 0.03
    # every final state has finite log density inside the cube
    assert np.all(np.isfinite(g["log_pi"])) and np.all((g["x"] >= 0) & (g["x"] <= 1))
    np.testing.assert_allclose(g["log_pi"], t.log_density(g["x"]), rtol=1e-4, atol=1e-2)


def test_generic_dimension_path():
    """D != 8 / K != 4 take the runtime-size kernels: f64 Philox vs oracle."""
    from oracle.abi import OracleMixConfig, mix_run
    from paper_2402_08273_b200.mix import MixTarget
    t = MixTarget.config2(9, dim=5, n_comp=3)
    kw = dict(strategy="ra-grid", grid_n=2, chains=100, seed=4, log_steps=8)
    o = mix_run(t, OracleMixConfig(steps=200, rng="philox", adapt_mode="pooled", **kw))
    gpu = gpu_run(t, 200, precision="f64", rng="philox", adapt_mode="pooled", **kw)
    assert_same(o, gpu)


def _sharded_mix_worker(rank, world, port, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2402_08273_b200.distributed import ShardedMix
        from paper_2402_08273_b200.mix import MixConfig, MixTarget
        torch.cuda.set_device(0)
        t = MixTarget.config2(2)
        sm = ShardedMix(t, MixConfig(strategy="ra-grid", grid_n=3, chains=999, seed=8, precision="f64",
                                     rng="philox", trace_enabled=True))
        sm.init_chains()
        sm.run(40)
        x, _ = sm.engine.state()
        lam, n, _, _ = sm.engine.regions()
        q.put((rank, sm.plan.offset, x, lam, n))
        sm.engine.close()
    finally:
        dist.destroy_process_group()


def test_sharded_mix_equals_single_handle():
    """configs[1] over two ranks (gloo, both on cuda:0; host-mediated exchange
    between steps, no kernel waits on another rank): chains and region lambdas
    equal the single-handle pooled run."""
    import socket
    import torch.multiprocessing as mp
    from paper_2402_08273_b200.mix import MixTarget
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_mix_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=300) for _ in range(2)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    t = MixTarget.config2(2)
    ref = gpu_run(t, 40, strategy="ra-grid", grid_n=3, chains=999, seed=8, precision="f64", rng="philox",
                  adapt_mode="pooled")
    x = np.concatenate([o[2] for o in out], axis=0)
    np.testing.assert_array_equal(x, ref["x"])
    for o in out:
        np.testing.assert_array_equal(o[3], ref["lambda_"])
        np.testing.assert_array_equal(o[4], ref["n"])


def test_autocorrelation_on_device():
    """Device autocorrelation_time of recorded chain series equals the checker
    (pinned to the reference's function) on the same series; series shorter
    than 1,000 steps report the reference's invalid_argument status."""
    from oracle.abi import np_autocorrelation_time
    from paper_2402_08273_b200.mix import MixConfig, MixEngine, MixTarget
    t = MixTarget.config2(0)
    for dim in (-1, 0):
        eng = MixEngine(t, MixConfig(strategy="global", chains=4096, seed=3, precision="f32", rng="philox",
                                     series_steps=3000, series_dim=dim))
        eng.init_chains()
        eng.run(500)
        _, _, _, st = eng.autocorrelation(0, 8)
        assert np.all(st == 3)
        eng.run(2500)
        tau, neff, s2, st = eng.autocorrelation(100, 64)
        ser = eng.series()
        eng.close()
        for i in range(64):
            r = np_autocorrelation_time(ser[100 + i])
            if r is None:
                assert st[i] == 3
                continue
            assert st[i] == 0
            np.testing.assert_allclose([tau[i], neff[i], s2[i]], r, rtol=1e-9)


@pytest.mark.parametrize("case", ["d1k1", "batch1", "lambda_floor", "ragged_block", "fixed_pcg_many"])
def test_edge_cases_match_oracle(case):
    """Edge cases of the controller / accept boundary, f64 vs the oracle
    (PCG32 + literal where the reference composition applies, else Philox +
    pooled): a 1-D single-component target (generic kernel path), L = 1
    (an update after every visit), a target acceptance the walk cannot reach
    (lambda pinned at lambda_min), a chain count that is not a multiple of the
    block size, and Fixed with many chains on the reference's own streams."""
    from oracle.abi import OracleMixConfig, mix_run
    from paper_2402_08273_b200.mix import MixTarget
    t = MixTarget.config2(6)
    kw = dict(strategy="global", chains=37, seed=13, log_steps=16)
    rng, mode, steps = "pcg32", "literal", 300
    if case == "d1k1":
        t = MixTarget(np.array([1.0]), np.array([[0.5]]), np.array([[[0.01]]]))
    elif case == "batch1":
        kw.update(batch_size=1)
    elif case == "lambda_floor":
        kw.update(target_acceptance=0.999, lambda_min=-12.0)
        steps = 600
    elif case == "ragged_block":
        kw.update(chains=1000 + 37, strategy="ra-grid", grid_n=5)
        rng, mode = "philox", "pooled"
    elif case == "fixed_pcg_many":
        kw.update(strategy="fixed", chains=3000, lambda_init=-7.5)
    o = mix_run(t, OracleMixConfig(steps=steps, rng=rng, adapt_mode=mode, **kw))
    g = gpu_run(t, steps, precision="f64", rng=rng, adapt_mode=mode, **kw)
    assert_same(o, g)
    if case == "lambda_floor":
        assert g["lambda_"][0] == -12.0
