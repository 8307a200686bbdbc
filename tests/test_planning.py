"""Pipeline IR: passes, variant space, validation and lowering on a
planning-only engine (the reference front end + our passes; no GPU)."""
import pytest

import harness
from paper_1709_00700_b200 import InvalidConfig, Unsupported
from paper_1709_00700_b200 import queries as Q

PROJ = "single_pass/sequential/branched"
AGG = "local_hash/sequential/branched/linear_probing/murmur/wg=16/ht=1"


def load(planner, tables):
    for t in tables:
        cols = t.columns()
        planner.put_table(t.name, cols)


def _planner(tables):
    from paper_1709_00700_b200 import Engine
    e = Engine(-1)
    load(e, tables)
    return e


@pytest.fixture
def micro():
    return _planner(harness.micro_tables(1000, 7))


@pytest.fixture
def tpch():
    return _planner(harness.bench_tables("tpch", 0.001, 42))


@pytest.fixture
def ssb():
    return _planner(harness.bench_tables("ssb", 0.001, 42))


def test_variant_space_exact_counts(micro):
    # SPEC.md:540 acceptance 1: 32 projection variants (4 single-pass), 896 aggregation
    assert micro.space_size(Q.LISTING1, 0) == (32, 4)
    assert micro.space_size(Q.LISTING8, 0) == (896, 0)
    cfgs = {micro.space_config(Q.LISTING1, 0, i) for i in range(32)}
    assert len(cfgs) == 32


def test_pipeline_partitioning(micro, ssb, tpch):
    assert micro.pipeline_count(Q.LISTING1) == 1
    assert micro.pipeline_count(Q.JOIN2) == 3  # two builds + probe (Fig. 2)
    assert ssb.pipeline_count(Q.SSB_Q41) == 5
    assert tpch.pipeline_count(Q.TPCH_Q3) == 3


def test_apply_variant_validates_clean(micro, ssb):
    for proj in ("single_pass/coalesced/predicated", "multi_pass/sequential/branched/tm=1024",
                 "single_pass/coalesced/branched/u=4"):
        for agg in (AGG, "global_hash/coalesced/predicated/cuckoo/multiply_shift/wg=256",
                    "local_hash/coalesced/branched/cuckoo/murmur/wg=1024/ht=64/u=2"):
            assert micro.validate(Q.JOIN2, f"{proj};{agg}") == ""
            assert ssb.validate(Q.SSB_Q41, f"{proj};{agg}") == ""


def test_invalid_configs_raise(micro):
    with pytest.raises(InvalidConfig):
        micro.validate(Q.LISTING1, "local_hash/coalesced/branched|x")
    with pytest.raises(InvalidConfig):  # strategy of the wrong pipeline kind
        micro.validate(Q.LISTING1, "local_hash/coalesced/branched/linear_probing/murmur/wg=16/ht=1|")
    with pytest.raises(InvalidConfig):
        micro.validate(Q.LISTING1, "multi_pass/coalesced/branched/tm=3;" + AGG)
    with pytest.raises(InvalidConfig):
        micro.validate(Q.LISTING1, "single_pass/coalesced/branched/u=3;" + AGG)


def test_lowering_q6(tpch):
    text = tpch.explain(Q.TPCH_Q6, f"{PROJ};{AGG}")
    lines = [l for l in text.splitlines() if not l.startswith("pipeline")]
    assert sum(l.startswith("FILTER") for l in lines) == 5
    assert sum(l.startswith("ARITH") for l in lines) == 1
    # sum + the hidden .rows count (planner_pipelines.cpp:484-493)
    assert [l.split()[1] for l in lines if l.startswith("AGG")] == ["sum", "count"]


def test_lowering_q1_value_numbering(tpch):
    text = tpch.explain(Q.TPCH_Q1, f"{PROJ};{AGG}")
    # the reference emits 6 ARITHMETIC ops and 11 aggregates;
    # value numbering shares (100-d), ep*(100-d) and identical SUM/COUNTs
    assert sum(l.startswith("ARITH") for l in text.splitlines()) == 4
    assert sum(l.startswith("AGG") for l in text.splitlines()) == 6
    assert sum(l.startswith("KEY") for l in text.splitlines()) == 2


def test_lowering_q3_payload_chain(tpch):
    text = tpch.explain(Q.TPCH_Q3, f"{PROJ};{AGG}")
    # customer probe key is o_custkey fetched through the orders probe's row id
    assert "PROBE t1 key payload(" in text and "@p0" in text
    assert text.count("SINK HASH_PUT") == 2 and "SINK HASH_AGGREGATE" in text


def test_cross_join_lowers_to_pair_table(micro):
    # CROSS_JOIN (planner_pipelines.cpp:337-352) is rewritten into a LOOP over
    # a pair table (engine.cpp rewrite_cross_joins) for explain, compile_check
    # and finalize as for execution
    sql = "select lo_quantity, p_size from part, lineorder where p_size < 2 and lo_quantity < 2"
    text = micro.explain(sql, f"{PROJ};{AGG}")
    assert "__cross" in text and "lineorder*part" in text
    report = micro.compile_check(sql, f"{PROJ};{AGG}")
    assert all(" ok " in l for l in report.splitlines() if l), report


@pytest.mark.parametrize("key", [k for k, _ in harness.BENCH])
def test_compiled_programs_build_for_sm100a(key):
    # the generated program policy of every pipeline compiles with NVRTC for
    # sm_100a (code generation is checked here; execution in test_gpu_parity)
    db_name = "ssb" if key.startswith("ssb") else "tpch"
    e = _planner(harness.bench_tables(db_name, 0.001, 42))
    sql = dict(harness.BENCH)[key]
    for cfg in (f"{PROJ};{AGG}",
                "multi_pass/coalesced/predicated/tm=1024;"
                "global_hash/coalesced/predicated/cuckoo/multiply_shift/wg=256"):
        report = e.compile_check(sql, cfg)
        lines = [l for l in report.splitlines() if l]
        assert len(lines) == e.pipeline_count(sql)
        assert all(" ok " in l for l in lines), report
