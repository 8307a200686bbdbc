"""Registers / spills / smem of the compiled programs of a query (NVRTC + ptxas -v, no GPU):
python tools/jit_regs.py <query> [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1709_00700_b200 import Engine  # noqa: E402
from paper_1709_00700_b200 import datagen as dg  # noqa: E402
from paper_1709_00700_b200 import queries as Q  # noqa: E402

q = sys.argv[1]
sql, tables, fact = Q.BENCH[q]
e = Engine(-1)
for t in tables:
    name, cols = dg.host_table(t, 0.001, 42)
    e.put_table(name, cols)
cfg = sys.argv[2] if len(sys.argv) > 2 else ""
print(e.compile_check(sql, cfg))
