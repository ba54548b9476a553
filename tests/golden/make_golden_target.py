"""Generate tests/golden/target/*.npz for the analytic-target harness
(BASELINE.json configs[1]) from the UNMODIFIED reference's controller, accept
rule, quantile and RNG (oracle/_ref ref_mix_run, oracle/ref_harness.cpp).

Run in the build container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden_target.py
Each fixture stores the target (weights, means, covariances), the config and
the reference composition's outputs: per-chain decision logs (a, flags) of the
first K steps, final states and log densities, region lambdas / update counts
/ tallies and the update-event trace.  The lockstep composition is
deterministic at any chain count (one thread records in chain order).
"""
from __future__ import annotations

import dataclasses
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.abi import OracleMixConfig, build, mix_run  # noqa: E402
from paper_2402_08273_b200.mix import MixTarget  # noqa: E402

CASES = [
    # name, target seed, config
    ("target_global_1c", 0, dict(strategy="global", chains=1, steps=3000, seed=3, log_steps=64)),
    ("target_ragrid_1c", 1, dict(strategy="ra-grid", grid_n=4, chains=1, steps=3000, seed=5,
                                 log_steps=64)),
    ("target_global_16c", 2, dict(strategy="global", chains=16, steps=400, seed=7, log_steps=32)),
    ("target_ragrid_16c", 0, dict(strategy="ra-grid", grid_n=3, chains=16, steps=400, seed=9,
                                  log_steps=32)),
    ("target_fixed_64c", 0, dict(strategy="fixed", chains=64, steps=200, seed=11, log_steps=32,
                                 lambda_init=-8.0)),
]


def main():
    build(reference=True)
    out_dir = os.path.join(HERE, "target")
    os.makedirs(out_dir, exist_ok=True)
    for name, tseed, kw in CASES:
        tgt = MixTarget.config2(tseed)
        cfg = OracleMixConfig(**kw)
        r = mix_run(tgt, cfg, reference=True)
        np.savez_compressed(
            os.path.join(out_dir, name + ".npz"),
            config=json.dumps(dataclasses.asdict(cfg)), weights=tgt.weights, means=tgt.means,
            covariances=tgt.covariances, x=r["x"], log_pi=r["log_pi"], log_a=r["log_a"],
            log_f=r["log_f"], lambda_=r["lambda_"], n=r["n"], tally_accept=r["tally_accept"],
            tally_visits=r["tally_visits"], trace=r["trace"],
            scalars=np.array([r["accepted"], r["acceptance_sum"]], np.float64))
        print(name, "acc=%.4f" % r["mean_acceptance"], "lambda=", np.round(r["lambda_"], 3)[:4],
              "trace", r["trace"].shape)


if __name__ == "__main__":
    main()
