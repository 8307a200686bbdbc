"""SASS of a query's compiled pipeline programs (NVRTC for sm_100a, no GPU):
  python tools/jit_sass.py <query> [pipeline] [config]
Writes the generated source + cubin to /tmp/hawk_jit/ (HAWK_JIT_DUMP) and
prints an opcode census of the chosen pipeline's kernel (default: terminal)."""
import collections
import glob
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
DUMP = "/tmp/hawk_jit"
os.makedirs(DUMP, exist_ok=True)
for f in glob.glob(DUMP + "/*"):
    os.remove(f)
os.environ["HAWK_JIT_DUMP"] = DUMP
import bench  # noqa: E402
from paper_1709_00700_b200 import Engine  # noqa: E402
from paper_1709_00700_b200 import datagen as dg  # noqa: E402
from paper_1709_00700_b200 import queries as Q  # noqa: E402

q = sys.argv[1]
pipe = int(sys.argv[2]) if len(sys.argv) > 2 else -1
cfg = sys.argv[3] if len(sys.argv) > 3 else bench.DEFAULT_CONFIG[q]
sql, tables, fact = Q.BENCH[q]
e = Engine(-1)
for t in tables:
    name, cols = dg.host_table(t, 0.001, 42)
    e.put_table(name, cols)
print(e.compile_check(sql, cfg))
cubins = sorted(glob.glob(DUMP + "/*.cubin"), key=os.path.getmtime)
cub = cubins[pipe]
sass = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
open(cub + ".sass", "w").write(sass)
ops = collections.Counter()
for line in sass.splitlines():
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if m:
        ops[m.group(2)] += 1
print(cub, sum(ops.values()), "instructions")
for k, v in ops.most_common(40):
    print(f"{v:6d} {k}")
print("memory / atomic opcodes:")
for k, v in sorted(ops.items()):
    if k.split(".")[0] in ("LDG", "STG", "LDS", "STS", "ATOM", "ATOMS", "ATOMG", "RED", "REDG", "REDS",
                           "UBLKCP", "SYNCS", "LDGSTS", "UTMALDG"):
        print(f"  {v:6d} {k}")
