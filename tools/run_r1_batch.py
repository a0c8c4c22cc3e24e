"""Round-1 library (tools/r1_pkg, git-ignored build of the round-1 tree) on the batch
ladder workload, for regression checks: python tools/run_r1_batch.py --qubits 24"""
import os
import runpy
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "r1_pkg"))
import paper_2511_19291_b200 as t  # noqa: E402  (the round-1 package)

t.OPT_PRODUCT_PREFIX = 9
_orig = t.State.set_option


def _set_option(self, opt, v):
    if opt == 9:  # no product prefix in round 1
        return None
    return _orig(self, opt, v)


t.State.set_option = _set_option
sys.argv = [os.path.join(HERE, "bench_batch.py")] + sys.argv[1:]
runpy.run_path(os.path.join(HERE, "bench_batch.py"), run_name="__main__")
