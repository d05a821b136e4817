#!/usr/bin/env python3
"""Search the Fig. 6 / Fig. 7 toy fixtures (SPEC acceptance 1-2) with
the ORACLE ONLY, and write them to tests/golden/fig6.json / fig7.json.

Fig. 6 ("prioritization_example"): five tasks released together,
serial unit-batch execution; EDF misses 2 (J4, J5), LUF misses 3 (J2, J4, J5),
EUDF/UP misses 1 (J2).  Integer execution times <= 10, deadlines <= 30.
Fig. 7 ("consolidate"): eight tasks, batch size 4; uncertainty-
oblivious EDF batching misses 4, uncertainty-aware consolidation misses 2.

Time unit: 1 "slot" = 1000 µs; latency = eta * len with eta = 1000 µs, no
setup/base; predictions exact (u = len).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

UNIT = 1000
BASEP = dict(eta_us=UNIT, mu_us=UNIT, base_us=0, setup_us=0, xi_us=0, **{"lambda": 1.5}, alpha=1.0, tau=1e9,
             u_max=10.0, C=1, b10=10, tightness=1, gamma=1, cores=1, policy="UP", consolidate=0, offload=0,
             raw_numerator=0)


def misses(lens, dls, n_per, prof):
    """lens, dls: [I, n] instance arrays -> misses per instance under prof (all via the oracle)."""
    I = lens.shape[0]
    u = lens.reshape(-1).astype(np.float32)
    D = (dls.reshape(-1) * UNIT).astype(np.uint32)
    k, _ = oracle.key(u, None, prof, r_us=np.zeros(len(u), np.int64), D_in=D)
    off = (np.arange(I + 1) * n_per).astype(np.uint32)
    st, _ = oracle.simulate(np.zeros(len(u), np.int64), lens.reshape(-1).astype(np.uint16), u, k, D, off, prof)
    return st["misses"]


def search(n, target, profs, rng, batch=20000, rounds=200):
    for _ in range(rounds):
        lens = rng.integers(1, 11, size=(batch, n))
        dls = rng.integers(1, 31, size=(batch, n))
        ok = np.ones(batch, bool)
        for name, want in target.items():
            ok &= misses(lens, dls, n, profs[name]) == want
        if ok.any():
            i = int(np.nonzero(ok)[0][0])
            return lens[i].tolist(), dls[i].tolist()
    raise SystemExit("no instance found")


def main():
    rng = np.random.default_rng(20230906)
    p6 = {k: dict(BASEP, policy=k) for k in ("EDF", "LUF", "UP")}
    lens, dls = search(5, {"EDF": 2, "LUF": 3, "UP": 1}, p6, rng)
    fig6 = {"_doc": "found by scripts/find_fixtures.py (oracle only); Fig. 6 P:251-266, S:628",
            "unit_us": UNIT, "len": lens, "deadline_units": dls, "profiles": p6,
            "misses": {"EDF": 2, "LUF": 3, "UP": 1}}
    p7 = {"oblivious": dict(BASEP, policy="EDF", C=4, b10=10, consolidate=0),
          "aware": dict(BASEP, policy="EDF", C=4, b10=20, consolidate=1)}
    lens, dls = search(8, {"oblivious": 4, "aware": 2}, p7, rng)
    fig7 = {"_doc": "found by scripts/find_fixtures.py (oracle only); Fig. 7 P:269-285, S:629",
            "unit_us": UNIT, "len": lens, "deadline_units": dls, "profiles": p7,
            "misses": {"oblivious": 4, "aware": 2}}
    for name, obj in (("fig6.json", fig6), ("fig7.json", fig7)):
        with open(os.path.join(ROOT, "tests", "golden", name), "w") as f:
            json.dump(obj, f, indent=1)
            f.write("\n")
        print(name, obj["len"], obj["deadline_units"])


if __name__ == "__main__":
    main()
