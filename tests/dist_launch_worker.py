"""Worker script for tests/test_dist_gloo.py::test_launch_ranks_gloo: started
by paper_2110_08321_b200.dist.launch_ranks (torch.distributed.run, the same
launcher bench.py --gpus N uses), it joins a gloo group from the launcher's
environment, all-reduces its rank, max-reduces a timing and all-gathers
per-rank words; rank 0 writes what it saw to the path in argv[1]."""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2110_08321_b200 import dist as D  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", init_method="env://")
    acc = torch.tensor([rank + 1], dtype=torch.int64)
    D.reduce_partials(acc, world)
    t = D.max_over_ranks(0.25 * (rank + 1))
    got = D.gather_outputs(torch.full((4,), 100 + rank, dtype=torch.int64), world)
    if rank == 0:
        with open(sys.argv[1], "w") as f:
            json.dump({"world": world, "sum": int(acc.item()), "tmax": t, "gathered": got.tolist(),
                       "master": os.environ["MASTER_ADDR"]}, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
