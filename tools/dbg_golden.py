import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from tests.test_golden import load
from paper_1704_06967_b200.solver import Handle
from tests._oracle import ORACLE
z, st, cfg = load("tiny_dso8")
for kind in ("ic", "fc"):
    g = getattr(Handle(st, "gpu"), f"{kind}_run")(cfg)
    o = getattr(Handle(st, ORACLE), f"{kind}_run")(cfg)
    print(kind, "gpu", [ "%.10e" % s.energy for s in g.iters])
    print(kind, "ora", [ "%.10e" % s.energy for s in o.iters])
    print(kind, "gold", [ "%.10e" % e for e in z[f"{kind}_energies"]])
    print(kind, "acc", [s.accepted for s in g.iters], [s.accepted for s in o.iters], "maxupd", ["%.3g"%s.max_update_px for s in g.iters])
