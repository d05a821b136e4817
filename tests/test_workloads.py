"""Host-side checks of the synthetic workloads the bench legs use (configs 4
and 5): shapes, seeding and the grouping invariants the legs rely
on.  No method arithmetic here (rtgen holds none)."""
import numpy as np

from rtgen import configs


def test_config5_grid_shape():
    pts = configs.config5_points()
    # 8 rate multipliers x tightness {1, 2} x 7 policies + 21 alpha + 21 b steps
    assert len(pts) == 8 * 2 * 7 + 21 + 21 == 154
    assert len({p["name"] + str(p["mult"]) for p in pts}) == 154
    assert sorted({p["mult"] for p in pts}) == sorted(configs.CONFIG5_MULTS)
    alphas = [p["overrides"]["alpha"] for p in pts if p["name"].startswith("alpha=")]
    assert np.allclose(alphas, np.arange(21) / 10)
    bs = [p["overrides"]["b10"] for p in pts if p["name"].startswith("b=")]
    assert bs == list(range(10, 31))
    base = [p for p in pts if "/t" in p["name"]]
    assert all(p["overrides"]["tightness"] in (1, 2) for p in base)
    # baselines run without consolidation and offloading, UP+C+O with both
    assert all(p["overrides"]["consolidate"] == 0 and p["overrides"]["offload"] == 0
               for p in base if p["name"].split("/")[0] in ("FIFO", "HPF", "LUF", "MUF", "UP"))
    assert all(p["overrides"]["consolidate"] == 1 and p["overrides"]["offload"] == 1
               for p in pts if p["name"].startswith("UP+C+O"))


def test_config5_arrivals_scale_with_rate():
    base = configs.config5_base(700, per_lm=2, per_trace=200)
    assert len(base["trace_off"]) == 9
    # LM blocks are contiguous (one scoring launch per LM regressor)
    assert list(base["trace_prof"]) == [0, 0, 1, 1, 2, 2, 3, 3]
    a1 = configs.config5_arrivals(base, 1.0)
    assert (a1 == base["arrival_us"]).all()  # multiplier 1 = the base ramp (same seed, same traces)
    per = 200
    spans = {}
    for m in (0.25, 1.0, 8.0):
        a = configs.config5_arrivals(base, m).reshape(-1, per)
        assert (np.diff(a, axis=1) >= 0).all()
        spans[m] = float(np.mean(a[:, -1] - a[:, 0]))
    assert spans[0.25] > spans[1.0] > spans[8.0]


def test_config4_grouped_is_a_reordering():
    a = configs.config4_shard(5, 512, n_traces=65536, per_trace=1024)           # 128 traces
    b = configs.config4_shard(5, 512, n_traces=65536, per_trace=1024, grouped=True)
    assert sorted(a["trace_ids"]) == sorted(b["trace_ids"])
    assert (np.diff(b["trace_prof"].astype(int)) >= 0).all()  # contiguous LM groups
    pos_a = {int(t): k for k, t in enumerate(a["trace_ids"])}
    per = 1024
    for k, t in enumerate(b["trace_ids"]):
        j = pos_a[int(t)]
        assert b["trace_prof"][k] == a["trace_prof"][j] == t % 4
        sa = slice(j * per, (j + 1) * per)
        sb = slice(k * per, (k + 1) * per)
        assert (a["arrival_us"][sa] == b["arrival_us"][sb]).all()
        assert (a["true_len"][sa] == b["true_len"][sb]).all()
        ta = a["data"][a["offsets"][j * per]:a["offsets"][(j + 1) * per]]
        tb = b["data"][b["offsets"][k * per]:b["offsets"][(k + 1) * per]]
        assert (ta == tb).all()


def test_traces_threads_do_not_change_data():
    a = configs.traces(3, range(100, 180), 50, lambda t: t % 4, threads=1)
    b = configs.traces(3, range(100, 180), 50, lambda t: t % 4, threads=8)
    for k in ("data", "offsets", "arrival_us", "true_len", "trace_off", "trace_prof"):
        assert (a[k] == b[k]).all(), k


def test_periodic_arrivals_definition():
    # r_{i+1} = r_i + D_i within each trace, r_0 = 0
    D = np.asarray([5, 7, 11, 2, 3, 4], np.uint32)
    r = configs.periodic_arrivals(np.asarray([0, 3, 3, 6], np.uint32), D)
    assert list(r) == [0, 5, 12, 0, 2, 5]


def test_variance_subsets_order_spread():
    rng = np.random.default_rng(3)
    u = rng.gamma(2.0, 10.0, 6000).astype(np.float32)
    sub = configs.variance_subsets(u, 1000)
    assert all(len(v) == 1000 and len(set(v.tolist())) == 1000 for v in sub.values())
    sd = {k: float(np.std(u[v])) for k, v in sub.items()}
    assert sd["small"] < sd["medium"] < sd["large"]
