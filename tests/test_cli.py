"""The command line (hawk-b200): commands, CSV / key-value
outputs and the exit-code contract (0 success, 1 verification failure,
2 usage error, 3 runtime / capacity error)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1709_00700_b200", "lib", "hawk-b200")
Q6 = ("select sum(l_extendedprice*l_discount) as revenue from lineitem where l_shipdate >= 19940101 "
      "and l_shipdate < 19950101 and l_discount >= 5 and l_discount <= 7 and l_quantity < 24")


def cli(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)


def test_usage_errors_exit_2():
    assert cli().returncode == 2
    assert cli("bogus").returncode == 2
    assert cli("run", "--sql").returncode == 2
    assert cli("emit-kernel", "--sql", "select from", "--db", "tpch").returncode == 2  # SyntaxError


def test_emit_kernel_needs_no_gpu():
    r = cli("emit-kernel", "--sql", Q6, "--db", "tpch", "--sf", "1",
            "--variant", "single_pass/coalesced/branched;global_hash/coalesced/predicated/cuckoo/murmur/wg=128")
    assert r.returncode == 0, r.stderr
    assert "struct JitProg" in r.stdout and "hk::pipeline_body<hk::JitProg" in r.stdout


def test_gen_writes_csv_the_reference_loads(tmp_path):
    from oracle_bridge import OraTable
    from paper_1709_00700_b200 import datagen as dg
    from paper_1709_00700_b200.engine import INT64, STRING
    r = cli("gen", "--db", "ssb", "--sf", "0.01", "--out", str(tmp_path))
    assert r.returncode == 0, r.stderr
    for t in (dg.DDATE, dg.SUPPLIER):
        name, cols = dg.SCHEMA[t]
        schema_lines = open(tmp_path / f"{name}.schema").read().split()
        schema = [(schema_lines[i], INT64 if schema_lines[i + 1] == "int64" else STRING)
                  for i in range(0, len(schema_lines), 2)]
        ref = OraTable.load_csv(str(tmp_path / f"{name}.csv"), name, schema)
        _, host = dg.host_table(t, 0.01, 42)
        for a, b in zip(ref.columns(), host):
            assert a.decoded() == b.decoded(), a.name


@pytest.mark.gpu
def test_run_from_csv_equals_generated_tables(tmp_path):
    assert cli("gen", "--db", "tpch", "--sf", "0.01", "--out", str(tmp_path)).returncode == 0
    a = cli("run", "--sql", Q6, "--data", str(tmp_path))
    b = cli("run", "--sql", Q6, "--db", "tpch", "--sf", "0.01")
    assert a.returncode == 0 and b.returncode == 0, (a.stderr, b.stderr)
    assert a.stdout == b.stdout and a.stdout.startswith("revenue\n")
    assert cli("run", "--sql", Q6, "--db", "tpch", "--sf", "0.01", "--expect-rows", "1").returncode == 0
    assert cli("run", "--sql", Q6, "--db", "tpch", "--sf", "0.01", "--expect-rows", "2").returncode == 1


@pytest.mark.gpu
def test_learn_explore_and_runtime_errors(tmp_path):
    conf, trace, csv = str(tmp_path / "l.conf"), str(tmp_path / "t.csv"), str(tmp_path / "e.csv")
    r = cli("learn", "--sql", Q6, "--db", "tpch", "--sf", "0.01", "--out", conf, "--trace", trace, "--reps", "1")
    assert r.returncode == 0, r.stderr
    assert "aggregation.strategy=" in open(conf).read()
    assert open(trace).readline().startswith("index,projection,aggregation,ms,status")
    r = cli("run", "--sql", Q6, "--db", "tpch", "--sf", "0.01", "--config", conf)
    assert r.returncode == 0, r.stderr
    r = cli("explore", "--sql", Q6, "--db", "tpch", "--sf", "0.01", "--kind", "projection", "--out", csv,
            "--reps", "1")
    assert r.returncode == 0, r.stderr
    assert len(open(csv).read().splitlines()) == 33
    # a runtime error (EmptyAggregate) exits 3
    r = cli("run", "--sql", "select min(l_quantity) from lineitem where l_quantity > 100", "--db", "tpch",
            "--sf", "0.01")
    assert r.returncode == 3 and "empty input" in r.stderr
