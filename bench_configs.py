"""bench_configs.py -- the other BASELINE.json configs on one B200 (bench.py
measures the headline config 2).  One JSON line per measured point.

  python bench_configs.py --config 0   # cfg-0 net, batch 1 (one inference's latency)
  python bench_configs.py --config 1   # HS matvec sweep, N=16384, one rescale
  python bench_configs.py --config 1 --method lola   # the LoLa comparators on the same grid
  python bench_configs.py --config 3   # CIFAR-shaped net, N=16384, 5 rescales
  python bench_configs.py --config 4 [--hs]  # conv layer sweep, N=16384 (torchrun: shard by output channel)
  python bench_configs.py --model ce --batch 8   # a reference builtin (cryptonets-hs / me / ce) or ce-mini
                                                 # through the general stage driver, B images per run

Device time with CUDA events on the engine's stream after warm-up; inputs are
fresh seeded encryptions (synthetic, BASELINE.json shapes/distributions).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DELTA = 2.0 ** 40


def timed(ctx, fn, steps, warmup):
    import torch
    stream = torch.cuda.ExternalStream(ctx.stream_ptr())
    for _ in range(warmup):
        fn()
    ctx.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


def config1(args):
    """BASELINE configs[1]: m x n in {64,256,1024,4096}^2, A ~ N(0,.05^2),
    v ~ U[-1,1]^n, N=16384, Q={60,40}, one rescale.  Reports rotations/s
    (key-switched, HS metering) and the HS kernel's achieved GB/s.  Under
    torchrun with --split-hs the kept diagonals are split over the ranks
    (per-rank extended-basis partial sums, one NCCL
    all-reduce, ModDown/rescale/folds on every rank; strong scaling)."""
    import torch
    import torch.distributed as dist
    from paper_2110_08321_b200 import dist as Dm
    from paper_2110_08321_b200 import hegpu as H
    from paper_2110_08321_b200.workloads import hs_sweep_case
    rank, world, local = _dist_env()
    split = args.split_hs and world > 1
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    ctx = H.Context(14, [45, 40], 45, seed=1, device=local)
    dims = [int(x) for x in args.dims.split(",")]
    for m in dims:
        for n in dims:
            A, x = hs_sweep_case(m, n)
            t0 = time.perf_counter()
            plan = ctx.hs_plan(A, 2)
            ctx.gen_rotation_keys(plan.rotations())
            setup_s = time.perf_counter() - t0
            for B in sorted({1, args.batch}):
                pt = ctx.encode(x, DELTA, 2)
                v = ctx.ct(B, 2, np.concatenate([ctx.encrypt(pt, 2, 7 + i) for i in range(B)]), DELTA)
                out = ctx.ct(B, 1)
                if split:
                    part = torch.empty(ctx.hs_acc_words(plan, B), dtype=torch.int64, device=f"cuda:{local}")

                    def run():
                        ctx.hs_matvec_partial(plan, v, rank, world, part)
                        ctx.sync()
                        Dm.reduce_partials(part, world)
                        ctx.hs_matvec_finish(plan, v, part, world, out)
                else:
                    def run():
                        ctx.hs_matvec(plan, v, out)
                run()  # first run fuses keys x masks (offline)
                ctx.reset_meter()
                run()
                tally = np.array(ctx.total(), dtype=np.int64)
                ms = Dm.max_over_ranks(timed(ctx, run, args.steps, args.warmup), device=f"cuda:{local}")
                if split:
                    tt = torch.tensor(tally, device=f"cuda:{local}")
                    dist.all_reduce(tt)
                    tally = tt.cpu().numpy()
                    tally[1] -= (world - 1) * B * plan.folds  # the folds run on every rank,
                    tally[4] -= (world - 1) * B * plan.folds  # the reference meters them once
                # correctness of every sweep point: the first image's decrypted
                # slots 0..m-1 against the cleartext A x (outside the timed runs)
                got = ctx.decode(ctx.decrypt(out.download()[: 2 * ctx.N], 1), 1, DELTA)[:m]
                err = float(np.abs(got - A @ x).max())
                assert err < 1e-4, f"config 1 m={m} n={n}: decrypted A x off by {err}"
                kms = kbytes = 0.0
                for kern in ("k_hs_diag", "k_hs_imma", "k_hs_narrow"):
                    ctx.kernel_timer(kern)
                    run()
                    a, _, b_ = ctx.kernel_timer_read()
                    kms, kbytes = kms + a, kbytes + b_
                ctx.kernel_timer(None)
                rot = int(tally[4])
                if rank == 0:
                    print(json.dumps({
                        "config": 1, "m": m, "n": n, "batch": B, "n_gpus": world,
                        "mode": "split-diagonals" if split else "single",
                        "ms_per_matvec_batch": ms,
                        "matvecs_per_s": B / (ms / 1e3), "rotations_per_s": rot / (ms / 1e3),
                        "rotations_per_matvec": rot // B, "mul_pc_per_matvec": int(tally[2]) // B,
                        "m_eff": plan.m_eff, "folds": plan.folds,
                        "hs_kernel_ms": kms, "hs_kernel_gbs": kbytes / (kms / 1e3) / 1e9 if kms else None,
                        "max_abs_err_vs_Ax": err,
                        "setup_s": setup_s}), flush=True)
            del plan
    if world > 1:
        dist.destroy_process_group()


def config1_lola(args):
    """The LoLa comparators of Fig. 2 on config 1's grid (measured, not
    predicted): lola_dense / lola_stacked (matvec.cpp:107-166) on one
    ciphertext (and a batch), N=16384, Q={60,40,40} (two rescales: product
    + the value-level clearing).  Reports rotations/s next to the metered
    counts, which equal predict_lola_* (matvec.cpp:189-211)."""
    from paper_2110_08321_b200 import hegpu as H
    from paper_2110_08321_b200.workloads import hs_sweep_case
    ctx = H.Context(14, [45, 40, 40], 45, seed=1)
    dims = [int(x) for x in args.dims.split(",")]
    for kind in ("dense", "stacked"):
        for m in dims:
            for n in dims:
                A, x = hs_sweep_case(m, n)
                try:
                    t0 = time.perf_counter()
                    plan = ctx.lola_plan(kind, A, 3)
                    ctx.gen_rotation_keys(plan.rotations())
                    setup_s = time.perf_counter() - t0
                except H.CapacityError as e:
                    print(json.dumps({"config": 1, "method": "lola-" + kind, "m": m, "n": n,
                                      "capacity_error": str(e)}), flush=True)
                    continue
                for B in sorted({1, args.batch}):
                    if B * plan.batches > 8192:  # products in flight (dense: m per input) at ~0.8 MB each
                        continue
                    pt = ctx.encode(x, DELTA, 3)
                    v = ctx.ct(B, 3, np.concatenate([ctx.encrypt(pt, 3, 7 + i) for i in range(B)]), DELTA)
                    out = ctx.ct(B * plan.per_input, 1)
                    ctx.reset_meter()
                    ctx.lola_matvec(plan, v, out)
                    tally = ctx.total()
                    ms = timed(ctx, lambda: ctx.lola_matvec(plan, v, out), args.steps, args.warmup)
                    print(json.dumps({
                        "config": 1, "method": "lola-" + kind, "m": m, "n": n, "batch": B,
                        "ms_per_matvec_batch": ms, "matvecs_per_s": B / (ms / 1e3),
                        "rotations_per_s": tally[4] / (ms / 1e3), "rotations_per_matvec": tally[4] // B,
                        "mul_pc_per_matvec": tally[2] // B, "setup_s": setup_s}), flush=True)
                del plan


def config0(args):
    """BASELINE configs[0]: the cfg-0 MNIST-sized net at batch 1 (latency of
    one encrypted inference, device-resident taps, one CUDA graph)."""
    args.batch = 1
    return config3(args, which=0)


def config3(args, which=3):
    """BASELINE configs[3]: CIFAR-shaped net (3x32x32 U[0,1], conv 5x5/2
    3->32, square, HS 6272->256, square, HS 256->10), N=16384, 5 rescales.
    Under torchrun: --split-hs splits HS1's diagonals across the ranks (same
    images on every rank, partial extended-basis sums all-reduced over NCCL,
    strong scaling); otherwise images are sharded (weak scaling)."""
    import torch
    import torch.distributed as dist
    from paper_2110_08321_b200 import dist as D
    from paper_2110_08321_b200 import hegpu as H
    from paper_2110_08321_b200.workloads import CFG0, CFG3, net_image, net_weights
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    cfg = CFG3 if which == 3 else CFG0
    ctx = H.Context(cfg.log_n, list(cfg.qbits), cfg.pbits, seed=which, device=local)
    t0 = time.perf_counter()
    net = H.Net(ctx, cfg, net_weights(cfg, which))
    setup_s = time.perf_counter() - t0
    B = args.batch
    split = args.split_hs or args.split_first
    first = 0 if split else rank * B
    taps = np.concatenate([net.encrypt_image(net_image(cfg, first + i), nonce=first + i) for i in range(B)])
    dt = ctx.ct(B * net.ntaps, net.top, taps, DELTA)
    out = ctx.ct(B, net.out_level)
    # --split-first: Conv1 + Flat1 by output map; --split-hs: HS1 by diagonal
    # range; both: two partial-sum all-reduces per step
    layer = (H.split_first_and_dense(0) if args.split_first and args.split_hs
             else H.SPLIT_FIRST_LAYER if args.split_first else 0)
    mode = {(True, False): "split-first", (False, True): "split-hs",
            (True, True): "split-first+hs"}.get((bool(args.split_first), bool(args.split_hs)), "image-shard")
    if split and world > 1:
        def run():
            net.run_split(dt, out, layer, rank, world, lambda t: D.reduce_partials(t, world))
        run()
        ref = ctx.ct(B, net.out_level)
        net.run(dt, ref)
        assert np.array_equal(out.download(), ref.download()), "split run differs from the single-GPU run"
        fn = run
        ctx.reset_meter()
        fn()
    else:
        net.run(dt, out)
        ctx.reset_meter()  # the capture meters one step (graph replays do not)
        fn = ctx.capture(lambda: net.run(dt, out))
    tally = ctx.total()
    if world > 1:
        dist.barrier()
    ms = timed(ctx, fn, args.steps, args.warmup)
    ms = D.max_over_ranks(ms, device=f"cuda:{local}")
    imgs = B if split else B * world
    if rank == 0:
        print(json.dumps({
            "config": which, "batch": B, "n_gpus": world, "mode": mode,
            "ms_per_step": ms, "inferences_per_s": imgs / (ms / 1e3),
            "rotations_per_s": tally[4] * (1 if split else world) / (ms / 1e3),
            "hops_per_inference": [t / B for t in tally], "setup_s": setup_s}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def builtin_program(args):
    """A reference builtin (proj/src/netcompile.cpp:567-628) through the
    general stage driver hegpu_prog: B encrypted images per run; ce runs at
    its declared n_slots = 16384 (N = 2^15, ~140 GB of keys and tables).
    The logits of every image are checked against the FP64 forward pass."""
    from paper_2110_08321_b200 import hegpu as H
    from paper_2110_08321_b200.workloads import BUILTIN_MODEL_JSON, model_forward
    m = H.Model.parse(BUILTIN_MODEL_JSON[args.model])
    model = {"name": args.model, "n_slots": m.n_slots, "in_c": m.in_c, "in_d": m.in_d}
    stages = m.lower()
    depth = sum(0 if s["kind"] == "merge" else 2 if s["policy"] == "lola-dense" and s["kind"] == "linear" else 1
                for s in stages)
    log_n = (2 * model["n_slots"]).bit_length() - 1
    t0 = time.perf_counter()
    ctx = H.Context(log_n, [45] + [40] * depth, 45, seed=11, device=0)
    rng = np.random.default_rng(5)
    flat = rng.normal(0, 0.05, m.weight_floats).astype(np.float32).astype(np.float64)
    prog = H.Program(ctx, m, flat)
    B = args.batch
    imgs = rng.uniform(0, 1, (B, model["in_c"], model["in_d"], model["in_d"]))
    cts = np.concatenate([prog.encrypt_input(imgs[b], nonce=b) for b in range(B)])
    din, out = ctx.ct(B * prog.input_cts, prog.top, cts, DELTA), ctx.ct(B, prog.out_level)
    prog.run(din, out)   # resolves the plans' fused key tables
    setup = time.perf_counter() - t0
    ctx.reset_meter()
    prog.run(din, out)
    rows = ctx.stages()
    total = ctx.total()
    ms = timed(ctx, lambda: prog.run(din, out), args.steps, args.warmup)
    got = out.download().reshape(B, -1)
    err = max(np.abs(prog.decrypt_logits(got[b]) - model_forward(m.layers, m.in_c, m.in_d, flat, imgs[b])).max()
              for b in range(B))
    assert err < 1e-3, err
    print(json.dumps({"model": model["name"], "n_slots": model["n_slots"], "log_n": log_n, "levels": depth + 1,
                      "batch": B, "ms_per_run": ms, "inferences_per_s": B / ms * 1e3,
                      "rotations_per_s": total[4] / ms * 1e3, "hops_per_inference": [v / B for v in total],
                      "stages": [r[0] for r in rows], "max_abs_logit_err": float(err), "setup_s": setup}))


def _dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def _ref_conv_map(img, w, b):
    """FP64 direct convolution of one output map (stride 1), the spot check"""
    c_in, d_in, _ = img.shape
    k = w.shape[-1]
    d_out = d_in - k + 1
    out = np.full((d_out, d_out), float(b))
    for ci in range(c_in):
        for ky in range(k):
            for kx in range(k):
                out += w[ci, ky, kx] * img[ci, ky: ky + d_out, kx: kx + d_out]
    return out.ravel()


def config4(args):
    """BASELINE configs[4]: conv-layer sweep, c_in in {1,3,16,32}, 32x32
    U[0,1] inputs, k in {3,5} (stride 1), c_out in {5,32,64}, N=16384,
    weights N(0,.05^2).  Conv-pack (convlower.cpp:39-74) sharded by output
    channel over the ranks of a torchrun job (no collective on the data
    path; the step time is the max over ranks), HOPs summed over ranks; and
    the Halevi-Shoup formulation of the same layer (conv_to_matrix +
    hs_matvec, convlower.cpp:76-102 / matvec.cpp:82-105) where it fits one
    ciphertext (the reference throws CapacityError elsewhere), its
    diagonals split over the ranks with an all-reduce of the partial sums."""
    import torch
    import torch.distributed as dist
    from paper_2110_08321_b200 import hegpu as H
    from paper_2110_08321_b200 import dist as Dm
    from paper_2110_08321_b200.workloads import conv_as_matrix, conv_pack_image
    rank, world, local = _dist_env()
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    ctx = H.Context(14, [45, 40], 45, seed=4, device=local)
    rng = np.random.default_rng(4)

    def tmax(ms):
        return Dm.max_over_ranks(ms, device=f"cuda:{local}")

    for c_in in (1, 3, 16, 32):
        img = rng.uniform(0, 1, (c_in, 32, 32))
        for k in (3, 5):
            d_out = 32 - k + 1
            ntaps = k * k * c_in
            taps = conv_pack_image(img, k)
            cts = np.concatenate([ctx.encrypt(ctx.encode(t, DELTA, 2), 2, i) for i, t in enumerate(taps)])
            dt = ctx.ct(ntaps, 2, cts, DELTA)
            for c_out in (5, 32, 64):
                W = rng.normal(0, 0.05, (c_out, c_in, k, k))
                b = rng.normal(0, 0.01, c_out)
                lo, hi = c_out * rank // world, c_out * (rank + 1) // world  # this rank's output channels
                line = {"config": 4, "c_in": c_in, "k": k, "c_out": c_out, "n_gpus": world,
                        "sharding": "output channels"}
                if hi > lo:
                    out = ctx.ct(hi - lo, 1)
                    plan = ctx.conv_plan(ntaps, W[lo:hi].reshape(hi - lo, -1), b[lo:hi], d_out * d_out, 2, DELTA)
                    ctx.reset_meter()
                    ctx.conv_plan_run(plan, dt, out)
                    tally = np.array(ctx.total(), dtype=np.int64)
                    ms = timed(ctx, lambda: ctx.conv_plan_run(plan, dt, out), args.steps, args.warmup)
                    err = 0.0
                    if rank == 0:  # spot check: map 0 against the FP64 direct conv
                        got = ctx.decode(ctx.decrypt(out.download()[: 2 * ctx.N], 1), 1, DELTA)[: d_out * d_out]
                        err = float(np.abs(got - _ref_conv_map(img, W[0], b[0])).max())
                else:
                    tally, ms, err = np.zeros(5, dtype=np.int64), 0.0, 0.0
                ms = tmax(ms)
                if world > 1:
                    tt = torch.tensor(tally, device=f"cuda:{local}")
                    dist.all_reduce(tt)
                    tally = tt.cpu().numpy()
                line.update({"ms_per_layer": ms, "layers_per_s": 1e3 / ms,
                             "hops": dict(zip(H.TALLY_FIELDS, [int(x) for x in tally])),
                             "max_abs_err_vs_ref_conv": err})
                if args.hs and c_in * 32 * 32 <= ctx.S:
                    line["hs"] = hs_formulation(ctx, W, b, img, world, rank, local, args)
                if rank == 0:
                    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def hs_formulation(ctx, W, b, img, world, rank, local, args):
    """the conv layer as one HS matvec (conv_to_matrix), if it fits"""
    import torch
    from paper_2110_08321_b200 import hegpu as H
    from paper_2110_08321_b200 import dist as Dm
    from paper_2110_08321_b200.workloads import conv_as_matrix
    A = conv_as_matrix(W, 32)
    try:
        t0 = time.perf_counter()
        plan = ctx.hs_plan(A, 2)
    except H.CapacityError as e:
        return {"capacity_error": str(e)}
    ctx.gen_rotation_keys(plan.rotations())
    setup_s = time.perf_counter() - t0
    x = img.ravel()
    v = ctx.ct(1, 2, ctx.encrypt(ctx.encode(x, DELTA, 2), 2, 99), DELTA)
    out = ctx.ct(1, 1)
    if world > 1:
        words = ctx.hs_acc_words(plan, 1)
        part = torch.empty(words, dtype=torch.int64, device=f"cuda:{local}")

        def run():
            ctx.hs_matvec_partial(plan, v, rank, world, part)
            ctx.sync()
            Dm.reduce_partials(part, world)
            ctx.hs_matvec_finish(plan, v, part, world, out)
    else:
        def run():
            ctx.hs_matvec(plan, v, out)
    ctx.reset_meter()
    run()
    tally = ctx.total()
    ms = Dm.max_over_ranks(timed(ctx, run, args.steps, args.warmup), device=f"cuda:{local}")
    rot = tally[4] if world == 1 else None
    res = {"m": A.shape[0], "n": A.shape[1], "m_eff": plan.m_eff, "kept_diagonals": plan.kept,
           "folds": plan.folds, "ms": ms, "setup_s": setup_s}
    if world == 1:
        res.update({"rotations": int(tally[4]), "mul_pc": int(tally[2]), "rotations_per_s": tally[4] / (ms / 1e3)})
        if rank == 0:
            want = A @ x + 0.0
            got = ctx.decode(ctx.decrypt(out.download(), 1), 1, DELTA)[: A.shape[0]]
            res["max_abs_err_vs_ref"] = float(np.abs(got - want).max())
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, choices=[0, 1, 3, 4])
    ap.add_argument("--model", choices=["cryptonets-hs", "me", "ce", "ce-mini"],
                    help="run a builtin model through the general stage driver instead of a config")
    ap.add_argument("--method", default="hs", choices=["hs", "lola"],
                    help="config 1: the HS matvec (default) or the two LoLa comparators")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--dims", default="64,256,1024,4096", help="config 1 matrix dims (m and n)")
    ap.add_argument("--split-first", action="store_true",
                    help="configs 0 / 3 under torchrun: split Conv1 + Flat1 by output map across ranks")
    ap.add_argument("--split-hs", action="store_true",
                    help="configs 1 / 3 under torchrun: split the (first) HS layer's diagonals across ranks")
    ap.add_argument("--hs", action="store_true",
                    help="config 4: also run the Halevi-Shoup formulation where it fits one ciphertext")
    args = ap.parse_args()
    if args.model:
        return builtin_program(args)
    if args.config is None:
        ap.error("--config or --model is required")
    if args.config == 1 and args.method == "lola":
        return config1_lola(args)
    {0: config0, 1: config1, 3: config3, 4: config4}[args.config](args)


if __name__ == "__main__":
    main()
