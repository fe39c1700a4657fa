"""parallel.build_table with real ranks: launched by torchrun with --nproc-per-node N, every rank on
the same visible GPU (the build box has one), collectives over gloo (NCCL refuses two ranks on one
device).  The ranks' kernels never wait on one another -- only the host-side all-reduces do -- so
sharing the GPU is safe.  Rank 0 checks the table against the single-process build_table bit for
bit, and the failing-cell error against the single-process message, then prints one JSON line.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \\
        tools/multirank_check.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    import paper_1305_6738_b200 as zk
    from paper_1305_6738_b200 import parallel

    grids = [dict(ns=(20, 300, 1500), gammas=(1.6, 2.4), support=zk.Support.unbounded(), base_seed=9, replicates=3001,
                  repetitions=2),
             dict(ns=(50, 700), gammas=(0.5, 1.5), support=zk.Support.finite(1000), base_seed=4, replicates=2000,
                  repetitions=1)]
    tables = [parallel.build_table(**kw) for kw in grids]
    fail = dict(ns=(3,), gammas=(1.0, -30.0), support=zk.Support.finite(20), base_seed=5, replicates=100,
                repetitions=2)
    try:
        parallel.build_table(**fail)
        multi_err = None
    except zk.SimulationError as err:
        multi_err = str(err)
    if rank == 0:
        same = [t.cells == zk.build_table(**kw).cells for t, kw in zip(tables, grids)]
        try:
            zk.build_table(**fail)
            single_err = None
        except zk.SimulationError as err:
            single_err = str(err)
        print(json.dumps({"world": world, "tables_bit_identical": same, "error_equal": multi_err == single_err,
                          "error": multi_err}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
