"""Algorithm 1 on CPU: the engine's
coordinate descent (engine/learner.cpp) driven through the C ABI with
synthetic costs instead of CUDA-event measurements."""
import ctypes as C
import math

import pytest

from paper_1709_00700_b200 import _native

# preferred value per workload dimension (SPEC.md:244-252 value lists)
PREFER = {
    "proj": "multi_pass", "agg": "local_hash", "tm": "tm=1024", "wg": "wg=64",
    "access": "coalesced", "ht": "ht=64", "pred": "predicated", "impl": "cuckoo",
    "fn": "multiply_shift",
}


def fields(config: str) -> dict:
    proj, agg = config.split(";")
    p, a = proj.split("/"), agg.split("/")
    f = {"proj": p[0], "agg": a[0], "access": a[1], "pred": a[2], "impl": a[3], "fn": a[4]}
    for part in p + a:
        for key in ("tm", "wg", "ht"):
            if part.startswith(key + "="):
                f[key] = part
    return f


def learn(cost, q=3, early=1, starts=None):
    lib = _native.engine()
    calls = []

    def cb(cfg, _user):
        calls.append(cfg.decode())
        return cost(cfg.decode())

    fn = _native.COST_FN(cb)
    best = C.create_string_buffer(512)
    ms, ev, sw = C.c_double(), C.c_int32(), C.c_int32()
    assert lib.hawk_learn_with_cost(fn, None, q, early, starts.encode() if starts else None, best,
                                    512, C.byref(ms), C.byref(ev), C.byref(sw)) == 0, \
        lib.hawk_engine_last_error()
    return best.value.decode(), ms.value, ev.value, sw.value, calls


def separable(cfg: str) -> float:
    f = fields(cfg)
    return 1.0 + sum(0.0 if f.get(k) == v else 1.0 for k, v in PREFER.items())


def test_separable_cost_reaches_optimum_in_one_sweep():
    best, ms, ev, sw, calls = learn(separable)
    f = fields(best)
    for k, v in PREFER.items():
        assert f.get(k) == v, (k, best)
    assert ms == 1.0
    assert sw == 2  # the second sweep changes nothing: early termination
    assert ev == len(calls) == len(set(calls))  # every configuration measured once (cache)


def test_ties_keep_the_current_value_and_q_bounds_sweeps():
    # flat cost: nothing ever beats the base configuration (strict <)
    best, ms, ev, sw, _ = learn(lambda cfg: 5.0, q=3)
    base, *_ = learn(lambda cfg: 5.0, q=1)
    assert best == base and ms == 5.0 and sw == 1
    # without early termination all q sweeps run
    *_, sw3, _ = learn(separable, q=3, early=0)
    assert sw3 == 3


def test_failed_variants_are_infinite():
    # variants that "fail" (inf) are never chosen
    def cost(cfg):
        f = fields(cfg)
        return math.inf if f["impl"] == "cuckoo" else separable(cfg)
    best, ms, *_ = learn(cost)
    assert fields(best)["impl"] == "linear_probing" and math.isfinite(ms)


B200_START = "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8"


def trap(cfg: str) -> float:
    """TPC-H Q1-like landscape: local_hash is pruned (inf) at small work
    groups, global_hash is slow everywhere, local_hash with wg >= 128 is fast."""
    f = fields(cfg)
    if f["agg"] == "global_hash":
        return 100.0
    wg = int(f["wg"].split("=")[1])
    return math.inf if wg < 128 else 1.0 + (0.0 if f.get("ht") == "ht=8" else 0.5)


def test_restart_escapes_a_pruned_region():
    # from the reference default (wg=16) the descent settles on global_hash ...
    best, ms, *_ = learn(trap)
    assert fields(best)["agg"] == "global_hash" and ms == 100.0
    # ... a second start in the fast region (shared cache) finds local_hash
    best2, ms2, *_ = learn(trap, starts="|".join([
        "single_pass/sequential/branched;local_hash/sequential/branched/linear_probing/murmur/wg=16/ht=1",
        B200_START]))
    assert fields(best2)["agg"] == "local_hash" and ms2 == 1.0


def descend(sizes, cost, q=3, early=1):
    lib = _native.engine()
    calls = []

    def cb(idx, n, _user):
        v = tuple(idx[i] for i in range(n))
        calls.append(v)
        return cost(v)

    fn = _native.INDEX_COST_FN(cb)
    n = len(sizes)
    arr = (C.c_int32 * n)(*sizes)
    best = (C.c_int32 * n)()
    ms, ev, sw, ev1 = C.c_double(), C.c_int32(), C.c_int32(), C.c_int32()
    assert lib.hawk_coordinate_descent(n, arr, fn, None, q, early, best, C.byref(ms), C.byref(ev),
                                       C.byref(sw), C.byref(ev1)) == 0, lib.hawk_engine_last_error()
    return tuple(best), ms.value, ev.value, sw.value, ev1.value, calls


def test_separable_472_space_spec_acceptance_5():
    # 3 dimensions x {4, 7, 2} values, separable cost: the
    # brute-force optimum in sweep 1 with <= 13 evaluations, then termination
    # by sweep 2 through the unchanged-configuration check (lines 19-21)
    import itertools
    pen = [[3.0, 1.0, 0.0, 2.0], [5.0, 4.0, 6.0, 0.5, 2.0, 3.0, 1.0], [1.0, 0.0]]
    cost = lambda v: sum(pen[d][v[d]] for d in range(3))  # noqa: E731
    brute = min(itertools.product(range(4), range(7), range(2)), key=cost)
    best, ms, ev, sw, ev1, calls = descend([4, 7, 2], cost)
    assert best == brute and ms == cost(brute)
    assert ev1 <= 13
    assert sw == 2
    assert ev == len(set(calls))


def test_q0_returns_the_base_configuration():
    best, ms, ev, sw, ev1, calls = descend([4, 7, 2], lambda v: 1.0, q=0)
    assert best == (0, 0, 0) and sw == 0


def test_config_file_round_trip(tmp_path):
    from paper_1709_00700_b200.engine import load_config, save_config
    cfg = ("multi_pass/coalesced/predicated/tm=1024/u=2;"
           "local_hash/sequential/branched/cuckoo/multiply_shift/wg=512/ht=64/u=4")
    path = str(tmp_path / "learned.conf")
    save_config(cfg, path)
    text = open(path).read()
    assert "projection.thread_multiplier=1024" in text and "aggregation.hash_table_impl=cuckoo" in text
    assert sum(1 for l in text.splitlines() if "=" in l and not l.startswith("#")) == 18
    assert load_config(path) == cfg
    # the whole-variant form loads too; bad keys and values are InvalidConfig
    (tmp_path / "b.conf").write_text("projection=single_pass/sequential/branched\n"
                                     "aggregation=global_hash/coalesced/branched/linear_probing/murmur/wg=64\n")
    assert load_config(str(tmp_path / "b.conf")).endswith("wg=64")
    from paper_1709_00700_b200 import InvalidConfig
    (tmp_path / "c.conf").write_text("aggregation.work_group_size=abc\n")
    with pytest.raises(InvalidConfig):
        load_config(str(tmp_path / "c.conf"))
