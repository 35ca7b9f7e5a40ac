"""World-size-2 gloo test of the multi-GPU host logic (image sharding,
output-ciphertext all-gather, max-over-ranks timing) on CPU."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_08321_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, per_rank, words, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    imgs = list(D.image_range(rank, per_rank))
    # stand-in output ciphertexts: deterministic words per global image index
    local = np.concatenate([np.full(words, 1000 + i, dtype=np.uint64) for i in imgs])
    got = D.gather_outputs(torch.from_numpy(local.view(np.int64)), world)
    t = D.max_over_ranks(0.5 + rank)
    if rank == 0:
        arr = got.numpy().view(np.uint64).reshape(world * per_rank, words)
        q.put((arr[:, 0].tolist(), t))
    dist.destroy_process_group()


def test_shard_and_gather_two_ranks():
    world, per_rank, words = 2, 3, 16
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, per_rank, words, q)) for r in range(world)]
    for p in procs:
        p.start()
    firsts, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert firsts == [1000 + i for i in range(world * per_rank)]  # rank-ordered, no overlap
    assert t == 1.5  # max over ranks


def _reduce_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(rank)
    # residues below a 60-bit prime, as the HS partial accumulators hold
    part = rng.integers(0, (1 << 60) - 93, 64, dtype=np.uint64)
    acc = torch.from_numpy(part.view(np.int64).copy())
    D.reduce_partials(acc, world)
    q.put((rank, part, acc.numpy().view(np.uint64).copy()))
    dist.destroy_process_group()


def test_reduce_partials_two_ranks():
    """the config-3 HS partial-sum reduction: an int64 SUM all-reduce of
    uint64 residues is the exact element-wise sum (< 2^63 for <= 8 parts)"""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_reduce_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts = {r: part for r, part, _ in res}
    want = [int(a) + int(b) for a, b in zip(parts[0], parts[1])]
    for _, _, got in res:
        assert [int(x) for x in got] == want


def test_image_ranges_partition_the_batch():
    seen = [i for r in range(4) for i in D.image_range(r, 64)]
    assert seen == list(range(256))


def test_launch_ranks_gloo(tmp_path):
    """the real host launcher (dist.launch_ranks, used by bench.py --gpus N
    without a torchrun environment): N processes under torch.distributed.run
    on 127.0.0.1, each joining the group from the environment it sets"""
    import os
    import sys
    out = tmp_path / "r.json"
    script = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dist_launch_worker.py")
    rc = D.launch_ranks(2, script, [str(out)], env={"NCCL_DEBUG": "WARN"}, timeout=300)
    assert rc == 0
    import json
    r = json.loads(out.read_text())
    assert r["world"] == 2 and r["sum"] == 3 and r["tmax"] == 0.5 and r["master"] == "127.0.0.1"
    assert r["gathered"] == [100] * 4 + [101] * 4
