"""Worker of tests/test_gpu_sharding.py::test_two_process_gloo_sharded_solve_matches_oracle (TEST
INFRASTRUCTURE): one rank of a point-sharded solve, launched by torch.distributed.run with the gloo
backend.  Both ranks share cuda:0; the exchange is staged through host memory, so neither rank's
kernels ever wait on the other's.  Rank 0 compares the merged report with the oracle's
single-process solve and writes the verdict to <out>/rank0.json."""
import json
import os
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1704_06967_b200 import scenes, sharding  # noqa: E402
from paper_1704_06967_b200.solver import Handle  # noqa: E402


def main():
    out = Path(sys.argv[1])
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    rank = dist.get_rank()
    sc = scenes.make_scene(scenes.baseline_config("C1"), device="cpu")
    st = sc.state
    cfg = sc.cfg.solver_config()
    res = {}
    for kind in ("ic", "fc"):
        rep = sharding.solve_distributed(st, cfg, kind)
        if rank == 0:
            from tests._helpers import assert_final_params_close
            from tests._oracle import ORACLE
            ro = getattr(Handle(st, ORACLE), f"{kind}_run")(cfg)
            ok = (rep.iterations == ro.iterations and [s.accepted for s in rep.iters] == [s.accepted for s in ro.iters]
                  and rep.hessian_factorizations == ro.hessian_factorizations
                  and all(abs(a.energy - b.energy) <= 1e-4 * abs(b.energy) for a, b in zip(rep.iters, ro.iters)))
            try:
                assert_final_params_close(rep, ro, 1e-4, st, kind, cfg)
                params = True
            except AssertionError as e:
                params = str(e)
            res[kind] = {"control_flow_and_energies": bool(ok), "params": params, "iterations": rep.iterations,
                         "world": dist.get_world_size(), "final_energy": rep.final_energy,
                         "oracle_final_energy": ro.final_energy,
                         "warnings_equal": list(rep.warnings) == list(ro.warnings)}
    if rank == 0:
        (out / "rank0.json").write_text(json.dumps(res))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
