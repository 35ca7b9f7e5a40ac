"""Two real ranks (two processes, torch.distributed over gloo) driving the
multi-GPU code paths on the one GPU this build has: each rank owns its own
hegpu context (same seed -> same keys), its kernels run independently, and
only the host-side collective connects them -- no rank's kernel waits on
another's.  The results must be bit-identical to the single-process run.

  * config 3's split: the first layer by output map and HS1
    by diagonal range, every partial summed by an all-reduce of the device
    accumulator (copied through the host for gloo);
  * config 2's image sharding: each rank evaluates its own images, the output
    ciphertexts are all-gathered (dist.gather_outputs).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2110_08321_b200 import dist as D
    from paper_2110_08321_b200 import hegpu as H
    from paper_2110_08321_b200.workloads import CFG0, net_image, net_weights
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = CFG0
        ctx = H.Context(cfg.log_n, list(cfg.qbits), cfg.pbits, seed=2024, device=0)
        net = H.Net(ctx, cfg, net_weights(cfg, 7))
        B = 2
        imgs = [net_image(cfg, 300 + s) for s in range(B)]
        taps = ctx.ct(B * net.tap_cts, net.top,
                      np.concatenate([net.encrypt_image(im, nonce=300 + s) for s, im in enumerate(imgs)]), 2.0 ** 40)

        def reduce(t):  # the NCCL all-reduce of the bench, here over gloo through the host
            h = t.cpu()
            D.reduce_partials(h, world)
            t.copy_(h.to(t.device))

        out = ctx.ct(B, net.out_level)
        net.run_split(taps, out, H.split_first_and_dense(0), rank, world, reduce)
        split = out.download()
        # image sharding: rank r evaluates image r, outputs all-gathered
        mine = ctx.ct(1, net.out_level)
        one = ctx.ct(net.tap_cts, net.top, net.encrypt_image(imgs[rank], nonce=300 + rank), 2.0 ** 40)
        net.run(one, mine)
        local = torch.from_numpy(mine.download().view(np.int64).copy())
        gathered = D.gather_outputs(local, world).numpy().view(np.uint64)
        ref = ctx.ct(B, net.out_level)
        net.run(taps, ref)
        q.put((rank, split, gathered, ref.download()))
    finally:
        dist.destroy_process_group()


def test_two_ranks_split_and_gather_bit_identical():
    import socket

    import torch.multiprocessing as mp
    world = 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, split, gathered, ref = q.get(timeout=600)
        res[r] = (split, gathered, ref)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = res[0][2]
    assert np.array_equal(res[1][2], ref)  # same keys / randomness on both contexts
    for r in range(world):
        split, gathered, _ = res[r]
        assert np.array_equal(split, ref), f"rank {r}: split run differs from the single-process run"
        assert np.array_equal(gathered, ref), f"rank {r}: gathered image shards differ"
