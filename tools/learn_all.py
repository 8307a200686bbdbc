"""Algorithm 1 on the B200 for every BASELINE query at its own scale factor
(run under gpurun): per query, the learned configuration as a key-value file
paper_1709_00700_b200/learned/<query>.conf (what bench.py runs by default)
and the measurement trace as CSV under profiles/learn_r02_<query>.csv.
  python tools/learn_all.py [queries...]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import bench  # noqa: E402
from paper_1709_00700_b200 import Engine  # noqa: E402
from paper_1709_00700_b200 import queries as Q  # noqa: E402

REF_DEFAULT = "single_pass/sequential/branched;local_hash/sequential/branched/linear_probing/murmur/wg=16/ht=1"
B200_START = "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8"


def main():
    queries = sys.argv[1:] or list(bench.DEFAULT_CONFIG)
    for q in queries:
        sf = bench.BASELINE_SF[q]
        e = Engine(0)
        e.set_option("jit", 1)
        bench.load_tables(e, q, sf, 42, 0, 1)
        t0 = time.time()
        # three starts sharing one measurement cache: the reference default,
        # the B200 start, and the hand-picked configuration of round 1
        r = e.learn_ex([Q.BENCH[q][0]], q=3, reps=5, unroll_pass=True,
                       starts=[REF_DEFAULT, B200_START, bench.DEFAULT_CONFIG[q]],
                       trace_csv=os.path.join(ROOT, "profiles", f"learn_r02_{q}.csv"),
                       config_path=os.path.join(ROOT, "paper_1709_00700_b200", "learned", f"{q}.conf"))
        r.update(query=q, sf=sf, seconds=time.time() - t0)
        print(json.dumps(r), flush=True)
        e.close()


if __name__ == "__main__":
    main()
