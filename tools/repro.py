import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import harness
from paper_1709_00700_b200 import Engine
cfg = sys.argv[1]
which = sys.argv[2] if len(sys.argv) > 2 else "tpch"
e = Engine(0)
tables = harness.bench_tables(which, 0.01, 42)
harness.load_engine(e, tables)
db = harness.oracle_db(tables)
for key, sql in harness.BENCH:
    if key.startswith("ssb") != (which == "ssb"):
        continue
    try:
        r = e.run(sql, cfg)
        print(key, "diff:", harness.compare(db.execute(sql), r))
    except Exception as ex:
        print(key, "ERROR", type(ex).__name__, ex)
