"""bench.py -- encrypted-inference throughput of the B200 CKKS engine.

Workload (BASELINE.json configs[2]): the config-0 MNIST-sized CryptoNets/
LoLa-shaped net on 64 independent seeded images per GPU, run with the
reference's stages (proj/src/netcompile.cpp:321-447): conv_pack -> 25 tap
ciphertexts per image -> conv_packed_forward + rescale (5 maps) -> merge_maps
(4 key-switched rotations) -> square -> HS 845->100 -> square -> HS 100->10;
CKKS N=8192, Delta=2^40, Q = 60+5x40 bits, P = 60 bits.  One "step" is one
pass of the whole encrypted network over the 64-image batch.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

--gpus N without a torchrun environment re-launches itself with N ranks
(one process per GPU, NCCL; paper_2110_08321_b200.dist.launch_ranks).

Device-timed `value`: the reference-layout taps resident in HBM (1.26 GB per
step > 126 MB L2, so no L2 flush is needed), the step replayed as one CUDA
graph, CUDA events on the engine's own stream, max over ranks.  `e2e`: the
serving loop through the C-ABI (hegpu_net_submit_host_compact) from pinned
host memory -- H2D of the step's compact taps (25 per image) and D2H of the
output ciphertexts inside the timed region.  `fused` reports the same two
numbers for the fused, region-packed first layer (HEGPU_FIRST_LAYER_FUSED,
DESIGN.md §4.1c), which is not the reference's algorithm.

--impl reference times the CPU restatement (oracle/, plain C, -O3
-march=native) evaluating the same 64-image batch across all host cores --
the reference `hesim` itself is a plaintext simulator without CKKS and cannot
be built here.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "encrypted inferences/sec + key-switched rotations/sec, % of HBM roofline"
KERNELS = ["k_hs_diag", "k_hs_imma", "k_hs_narrow", "k_drop_ntt", "k_md_ntt", "k_md_intt", "k_ks_modup", "k_conv_mac", "k_intt_rows",
           "k_ks_intt", "k_ks_inner", "k_ntt_rows", "k_merge_c", "k_expand_c0", "k_expand_a", "k_wire_to_slot",
           "k_add", "k_tensor_square", "k_add_plain"]
NTT_KERNELS = ("k_drop_ntt", "k_md_ntt", "k_md_intt", "k_ks_modup", "k_intt_rows", "k_ks_intt", "k_ntt_rows")
UNIT = "inferences/s"
SEED = 2110
WORKLOAD = ("cfg2: 64 x cfg0 MNIST-sized net per GPU, reference stages (conv-pack 25 tap cts -> conv + rescale "
            "-> merge 5 maps (4 key-switched rotations) -> square -> HS 845->100 -> square -> HS 100->10), "
            "CKKS N=8192 L=6")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# IMAD.WIDE.U32 issue rate measured on B200 (tools/ubench_int.cu,
# profiles/r01_int_ubench.txt); one split-30/31 64x64 multiply-accumulate
# term is 4 IMAD.WIDE.U32
IMAD_WIDE_PER_CLK_SM = 59.0
N_SM = 148

# integer-pipe cost of one algorithmic op per kernel: a split-31 modular
# multiply-accumulate term is 4 IMAD.WIDE.U32; an NTT
# butterfly's Shoup product is 6 multiply instructions (modarith.cuh
# shoup_mul_lazy4) -- the ceiling if nothing but the multiplies issued
INT_OPS_IMAD = {"k_hs_diag": 4, "k_hs_narrow": 4, "k_ks_inner": 4, "k_drop_ntt": 6, "k_md_ntt": 6, "k_md_intt": 6,
                "k_ks_modup": 6,
                "k_intt_rows": 6, "k_ks_intt": 6, "k_ntt_rows": 6}
# kernels whose MACs run on the tensor cores (tcgen05.mma.kind::i8,
# conv_tc.cu / hs_tc.cu) as 64 byte-plane products each
TENSOR_KERNELS = ("k_hs_imma", "k_conv_mac")
TC_I8_POPS = 4.5  # nominal dense int8 tcgen05 rate of a B200 (2 ops per MAC)
# the NTT-family kernels run every butterfly of the 40/45-bit benchmark
# primes on the FP64 pipe: 6 FP64 instructions per product
# + 2 adds; B200 FP64 = 64 FMA lanes / clk / SM (half the FP32 rate)
NTT_FP64_KERNELS = ("k_drop_ntt", "k_md_ntt", "k_md_intt", "k_ks_modup", "k_intt_rows", "k_ks_intt", "k_ntt_rows")
FP64_PER_CLK_SM = 64.0
FP64_OPS_PER_BUTTERFLY = 8


def int_pipe_roofline(name, kd, clk_mhz):
    if not kd.get("modmuls"):
        return None
    if name in TENSOR_KERNELS:
        ops = kd["modmuls"] * 64 * 2 / (kd["ms_per_step"] / 1e3) / 1e12
        return {"pipe": "tensor (tcgen05 i8)", "achieved": ops, "peak": TC_I8_POPS * 1e3, "unit": "TOPS (byte-plane)",
                "frac": ops / (TC_I8_POPS * 1e3),
                "peak_basis": "nominal B200 dense int8 tcgen05 rate; 64 byte-plane MACs per modular MAC (useful work "
                              "only: band / plane padding excluded)"}
    if name in NTT_FP64_KERNELS:
        peak = N_SM * FP64_PER_CLK_SM * clk_mhz * 1e6 / FP64_OPS_PER_BUTTERFLY / 1e9
        return {"pipe": "fp64", "achieved": kd["gmodmul_s"], "peak": peak, "unit": "G butterflies/s",
                "frac": kd["gmodmul_s"] / peak,
                "peak_basis": f"{N_SM} SMs x {FP64_PER_CLK_SM:.0f} FP64/clk/SM x {clk_mhz:.0f} MHz / "
                              f"{FP64_OPS_PER_BUTTERFLY} FP64 instructions per butterfly"}
    per = INT_OPS_IMAD.get(name, 4)
    peak = N_SM * IMAD_WIDE_PER_CLK_SM * clk_mhz * 1e6 / per / 1e9
    return {"pipe": "int (IMAD)", "achieved": kd["gmodmul_s"], "peak": peak,
            "unit": "Gmodmul/s" if per == 4 else "G butterflies/s", "frac": kd["gmodmul_s"] / peak,
            "peak_basis": f"{N_SM} SMs x {IMAD_WIDE_PER_CLK_SM} IMAD.WIDE.U32/clk/SM x {clk_mhz:.0f} MHz / {per}"}


def ncu_traffic(kernel, launches):
    """dram__bytes_read.sum + dram__bytes_write.sum of `kernel` over one step
    (the newest committed ncu capture, profiles/), per launch of the timer
    run's `launches` per step (the ncu'd step runs as two 32-image parts, so
    it has twice the launches at half the rows each), or None"""
    for name in ("r02_traffic_step.json", "r01_traffic_step.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                t = json.load(f)
            return float(t[kernel]["dram_bytes"]) / max(1, launches), name
        except Exception:
            continue
    return None, None


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, every 10 ms) during the
    timed region; falls back to one nvidia-smi query if NVML is missing."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, device):
        self.device, self.rows, self._stop = device, [], threading.Event()

    def _run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((sm, mx, rs))
                self._stop.wait(0.01)
        except Exception:
            try:
                r = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm",
                                    "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10)
                sm, mx = [float(x) for x in r.stdout.strip().split(",")[:2]]
                self.rows.append((sm, mx, 0))
            except Exception:
                pass

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        time.sleep(0.02)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=10)

    def summary(self):
        sm = [r[0] for r in self.rows]
        mx = [r[1] for r in self.rows]
        reasons = sorted({name for r in self.rows for bit, name in self.REASONS.items() if r[2] & bit})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": float(max(mx)) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# --------------------------------------------------------------------------- CPU
def _cpu_prepare(images):
    """oracle state for the reference algorithm + the client's taps of `images`"""
    from oracle import ckks_pipeline as P
    from oracle.ckks import Ckks
    from paper_2110_08321_b200.workloads import CFG0, net_image, net_weights
    cfg = CFG0
    ck = Ckks(cfg.log_n, list(cfg.qbits), cfg.pbits, seed=SEED)
    # the reference's algorithm (per-map conv + rescale + merge), as the GPU arm
    prep = P.PreparedNet(ck, cfg, net_weights(cfg, SEED), merged=False)
    taps = [P.conv_pack_taps(ck, cfg, net_image(cfg, i), i, prep.tap_scale, merged=False) for i in images]
    return prep, taps


def _cpu_pool_worker(rank, nproc, n_images, steps, barrier, q):
    prep, taps = _cpu_prepare([i for i in range(n_images) if i % nproc == rank])
    for s in range(steps):
        barrier.wait()
        t0 = time.perf_counter()
        for t in taps:
            prep.eval(t)
        q.put((s, rank, time.perf_counter() - t0))


def cpu_batch_throughput(cores, n_images, steps):
    """the CPU port evaluating an `n_images` batch on `cores` processes
    (images dealt round-robin, keys / masks / taps prepared before the timed
    region, every step starting at a barrier): per step, inferences/s =
    n_images / the slowest process's evaluation time"""
    if cores == 1:
        prep, taps = _cpu_prepare(range(n_images))
        vals = []
        for _ in range(steps):
            t0 = time.perf_counter()
            for t in taps:
                prep.eval(t)
            vals.append(n_images / (time.perf_counter() - t0))
        return vals, f"{n_images} cfg0 image(s) evaluated on 1 core per step, keys/masks/taps prepared offline"
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    barrier, q = ctx.Barrier(cores), ctx.Queue()
    procs = [ctx.Process(target=_cpu_pool_worker, args=(r, cores, n_images, steps, barrier, q)) for r in range(cores)]
    for p in procs:
        p.start()
    res = [q.get() for _ in range(cores * steps)]
    for p in procs:
        p.join()
    per_step = {}
    for s, _, dt in res:
        per_step[s] = max(per_step.get(s, 0.0), dt)
    vals = [n_images / per_step[s] for s in sorted(per_step)]
    return vals, (f"{n_images} cfg0 images per step dealt over {cores} processes (one per host core), "
                  f"step time = slowest process; keys/masks/taps prepared before timing")


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import ckks
    ckks.use_native()  # -march=native build of the port, compiled on this host
    cores = os.cpu_count() or 1
    steps = max(1, args.steps)
    vals, sample = cpu_batch_throughput(cores, args.batch, steps + max(0, min(args.warmup, 1)))
    vals = vals[-steps:]  # the first step warms page cache / allocator when warmup > 0
    v = float(np.median(vals))
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 0, "steps": steps, "warmup": args.warmup,
            "ms_per_step": args.batch * 1e3 / v, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u64 (RNS mod q)", "data": "synthetic (seeded U[0,1] images, N(0,0.05^2) f32 weights)",
            "config": {"workload": WORKLOAD, "global_batch": args.batch, "parallelism": f"{cores} host processes"},
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU
def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2110_08321_b200 import dist as D
    from paper_2110_08321_b200 import hegpu as H
    from paper_2110_08321_b200.workloads import CFG0, net_image, net_weights, plain_forward

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    cfg = CFG0
    B = args.batch
    weights = net_weights(cfg, SEED)
    ctx = H.Context(cfg.log_n, list(cfg.qbits), cfg.pbits, seed=SEED, device=local)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=local)
    hbm, which = peaks()
    images = {i: net_image(cfg, i) for i in D.image_range(rank, B)}

    def timed(fn, steps):
        """device time per call of fn over `steps` calls, max over ranks"""
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return D.max_over_ranks(e0.elapsed_time(e1) / steps, device=dev)

    def measure(first_layer, detail):
        net = H.Net(ctx, cfg, weights, first_layer=first_layer)
        # client side (outside the timed region): conv-pack + encrypt this rank's images
        taps = np.concatenate([net.encrypt_image(images[i], nonce=i) for i in images])
        compact = np.concatenate([net.encrypt_image_compact(images[i], nonce=i) for i in images])
        dtaps = ctx.ct(B * net.tap_cts, net.top, taps, 2.0 ** 40)
        out = ctx.ct(B, net.out_level)
        gather_buf = torch.empty(B * net.out_words, dtype=torch.int64, device=dev)
        gathered = torch.empty(world * B * net.out_words, dtype=torch.int64, device=dev) if world > 1 else None
        for _ in range(args.warmup):
            net.run(dtaps, out)
        ctx.sync()
        # one step's HOP tally, executed key-switch work and kernel launches
        ctx.reset_meter()
        l0 = ctx.launches()
        graph = ctx.capture(lambda: net.run(dtaps, out)) if args.graph else None
        if graph is None:
            net.run(dtaps, out)
        ctx.sync()
        launches_per_step = ctx.launches() - l0
        tally, ks = ctx.total(), ctx.ks_counters()

        def step():
            if graph is not None:
                graph()
            else:
                net.run(dtaps, out)
            if world > 1:  # NCCL all-gather of the output ciphertexts (config 2)
                out.export_device(gather_buf.data_ptr())
                with torch.cuda.stream(stream):
                    D.gather_outputs(gather_buf, world, gathered)

        for _ in range(2):
            step()
        with ClockSampler(local) as clk:
            ms = timed(step, args.steps)
        host_out = out.download()
        # sanity (outside timing): decrypted logits of this rank's first image
        # against the cleartext network
        i0 = next(iter(images))
        logits = net.decrypt_logits(host_out[: net.out_words])
        err = float(np.abs(logits - plain_forward(cfg, weights, images[i0])).max())
        assert err < 1e-3, f"{first_layer}: decrypted logits off by {err}"

        # e2e through the public C-ABI from pinned host buffers: the client's
        # compact taps (c0 byte-packed + a-stream keys) go H2D in sub-chunks
        # overlapped with compute; outputs come back D2H
        pin_in = torch.from_numpy(compact).pin_memory()
        pin_out = torch.empty(B * net.out_words, dtype=torch.int64).pin_memory()

        def serve_step():  # step k+1's uploads overlap step k's compute
            net.submit_host_compact(pin_in, B, pin_out, args.chunk)

        for _ in range(max(4, args.warmup)):  # both staging buffers: direct, then captured
            serve_step()
        net.wait()
        e2e_ms = timed(serve_step, args.steps)
        net.wait()
        assert np.array_equal(pin_out.numpy().view(np.uint64), host_out), "e2e output differs from device run"
        res = {"ms": ms, "value": B * world / (ms / 1e3), "e2e_ms": e2e_ms,
               "e2e_value": B * world / (e2e_ms / 1e3), "h2d": int(compact.nbytes), "d2h": int(host_out.nbytes),
               "tally": tally, "ks": ks, "launches_per_step": launches_per_step, "clk": clk.summary(),
               "logit_err": err, "tap_cts": net.tap_cts, "compact_bytes": int(compact.nbytes),
               "full_bytes": int(taps.nbytes)}
        if detail:
            res["e2e_sync_ms"] = timed(lambda: net.run_host_compact(pin_in, B, pin_out, args.sync_chunk),
                                       max(2, args.steps // 2))
            # ---- per-kernel device time (CUDA events around every launch of
            # one kernel, one extra direct-launch step per kernel) -> roofline
            kernels = {}
            for name in KERNELS:
                ctx.kernel_timer(name)
                net.run(dtaps, out)
                kms, kn, kbytes, kops = ctx.kernel_timer_read_ops()
                if kn:
                    kernels[name] = {"ms_per_step": kms, "launches": kn, "alg_bytes": kbytes,
                                     "gbs": kbytes / (kms / 1e3) / 1e9 if kms > 0 else None,
                                     "modmuls": kops, "gmodmul_s": kops / (kms / 1e3) / 1e9 if kms > 0 else None,
                                     "share": kms / ms}
            ctx.kernel_timer(None)
            res["kernels"] = kernels
        del graph, dtaps, out, net
        ctx.sync()
        return res

    ref = measure("reference", True)
    fused = measure("fused", False) if not args.no_fused else None

    kernels = ref["kernels"]
    clk_mhz = ref["clk"]["sm_mhz"] or 1965.0
    for name, kd in kernels.items():
        kd["compute_roofline"] = int_pipe_roofline(name, kd, clk_mhz)
    dom = max(kernels, key=lambda k: kernels[k]["ms_per_step"])
    kd = kernels[dom]
    traffic, traffic_src = ncu_traffic(dom, kd["launches"])
    ms_max = ref["ms"]
    sec = ms_max / 1e3
    ntt_rows = sum(kernels[k]["modmuls"] for k in NTT_KERNELS if k in kernels) / ((1 << (cfg.log_n - 1)) * cfg.log_n)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": kd["gbs"], "peak": hbm, "unit": "GB/s",
                "frac": kd["gbs"] / hbm, "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": which,
                "alg_bytes_per_launch": kd["alg_bytes"] / kd["launches"],
                "avg_launch_ms": kd["ms_per_step"] / kd["launches"], "launches_per_step": kd["launches"],
                "share_of_step": kd["share"],
                # the NTT-family kernels are bound by the 64-bit multiply issue
                # rate more than HBM: their integer-pipe roofline
                "compute": int_pipe_roofline(dom, kd, clk_mhz),
                "note": "alg bytes / modmuls per launch per DESIGN.md §5 (LAUNCH_B byte models at each launch "
                        "site); achieved = alg bytes / summed CUDA-event launch time on the engine stream; "
                        "traffic = ncu dram bytes of the kernel over one step (profiles/) / launches_per_step"}
    tally, ks = ref["tally"], ref["ks"]
    line = {
        "metric": METRIC, "value": ref["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64 (RNS mod q, 60/40-bit primes)",
        "data": "synthetic (seeded U[0,1] 28x28 images padded to 29x29, N(0,0.05^2) f32 weights)",
        "config": {"workload": WORKLOAD, "first_layer": "reference", "global_batch": B * world,
                   "images_per_gpu": B, "parallelism": f"dp{world} (image sharding, NCCL all-gather of outputs)",
                   "tap_cts_per_image": ref["tap_cts"],
                   "l2": (f"device-resident inputs {ref['full_bytes'] / 1e9:.2f} GB of full tap ciphertexts per "
                          f"step (> 126 MB L2): no flush needed; e2e H2D {ref['compact_bytes'] / 1e6:.0f} MB "
                          f"compact taps per step")},
        # reference HOP semantics: hesim's per-stage tally (120 rotations +
        # 2 relinearisations per cfg-0 inference)
        "rotations_per_s": tally[4] * world / sec,
        "keyswitches_per_s": (tally[4] + tally[3]) * world / sec,
        "rotation_metering": "reference HOP semantics (hesim per-stage OpTally); see `performed` for the "
                             "key-switch work actually executed (hoisted HS diagonals share one ModUp)",
        "performed": {"per_step": ks, "modups_per_s": ks["modups"] * world / sec,
                      "key_inner_products_per_s": ks["key_inner_products"] * world / sec,
                      "moddowns_per_s": ks["moddowns"] * world / sec,
                      "rescales_per_s": ks["rescales"] * world / sec},
        # limb transforms per second: every NTT-family launch's butterflies
        # / (N/2 log2 N) (one transform = one limb of one polynomial)
        "ntts_per_s": ntt_rows * world / sec, "ntts_per_step": ntt_rows,
        "hops_per_inference": {k: v / B for k, v in zip(H.TALLY_FIELDS, tally)},
        "cuda_graph": bool(args.graph),
        "step_streams": (int(os.environ.get("HEGPU_NET_STREAMS", "2")) if B >= 64 else 1),
        "gpu_launches": ref["launches_per_step"] * args.steps,
        "roofline": roofline,
        "kernels": kernels,
        "clocks": ref["clk"],
        "e2e": {"value": ref["e2e_value"], "unit": UNIT, "h2d_bytes_per_step": ref["h2d"] * world,
                "d2h_bytes_per_step": ref["d2h"] * world, "ms_per_step": ref["e2e_ms"],
                "path": "hegpu_net_submit_host_compact per step (25 compact tap cts per image; step k+1 H2D "
                        "overlaps step k compute), timed to the last step's outputs on the host",
                "chunk": args.chunk},
        "e2e_sync": {"value": B * world / (ref["e2e_sync_ms"] / 1e3), "unit": UNIT, "ms_per_step": ref["e2e_sync_ms"],
                     "path": "hegpu_net_run_host_compact (one blocking call per step)", "chunk": args.sync_chunk},
        "logit_max_abs_err": ref["logit_err"],
        "peak_hbm_gbs": hbm, "peak_source": which,
    }
    if fused is not None:
        fsec = fused["ms"] / 1e3
        line["fused"] = {
            "note": "Conv1 + Flat1 fused by client-side replicated, region-packed taps (HEGPU_FIRST_LAYER_FUSED, "
                    "DESIGN.md §4.1c) -- not the reference's first-layer algorithm; same HOP tally",
            "value": fused["value"], "unit": UNIT, "ms_per_step": fused["ms"], "tap_cts_per_image": fused["tap_cts"],
            "e2e": {"value": fused["e2e_value"], "unit": UNIT, "ms_per_step": fused["e2e_ms"],
                    "h2d_bytes_per_step": fused["h2d"] * world, "d2h_bytes_per_step": fused["d2h"] * world},
            "performed_per_step": fused["ks"], "gpu_launches_per_step": fused["launches_per_step"],
            "rotations_per_s": fused["tally"][4] * world / fsec, "clocks": fused["clk"],
            "logit_max_abs_err": fused["logit_err"]}
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import ckks
        ckks.use_native()
        vals, sample = cpu_batch_throughput(1, args.cpu_images, 1)
        line["cpu_baseline"] = {"value": vals[0], "unit": UNIT, "cores": 1, "kind": "port", "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hegpu", choices=["hegpu", "reference"])
    ap.add_argument("--batch", type=int, default=64, help="images per GPU")
    ap.add_argument("--cpu-images", type=int, default=24, help="images in the 1-core cpu_baseline sample")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fused", action="store_true", help="skip the fused-first-layer extra measurement")
    ap.add_argument("--chunk", type=int, default=64, help="images per compute chunk in the pipelined e2e loop")
    ap.add_argument("--sync-chunk", type=int, default=32, help="images per chunk in the blocking e2e call")
    ap.add_argument("--graph", type=int, default=1, help="replay the device step as one CUDA graph")
    args = ap.parse_args()
    rank, world, _ = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl != "reference":
        # one process per GPU: re-launch under torch.distributed.run
        from paper_2110_08321_b200.dist import launch_ranks
        sys.exit(launch_ranks(args.gpus, os.path.abspath(__file__), sys.argv[1:]))
    if "WORLD_SIZE" in os.environ and world != args.gpus and args.impl != "reference":
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
