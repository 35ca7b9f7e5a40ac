"""bench.py -- encrypted-inference throughput of the B200 CKKS engine.

Workload (BASELINE.json configs[2]): the config-0 MNIST-sized CryptoNets/
LoLa-shaped net (conv 5x5/2 -> 5 maps via conv-packing, square, HS dense
845->100, square, HS dense 100->10; CKKS N=8192, Delta=2^40, Q = 60+5x40
bits, P = 60 bits) on 64 independent seeded images per GPU.  One "step" is
one pass of the whole encrypted network over the 64-image batch.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Device-timed value: taps resident in HBM (1.26 GB per step > 126 MB L2, so
no L2 flush is needed), CUDA events on the engine's own stream, max over
ranks.  e2e: the same step through hegpu_net_run_host from pinned host
buffers, both copies inside the timed region.  --impl reference times the
CPU restatement (oracle/, plain C, one image per host core) -- the
reference `hesim` itself is a plaintext simulator without CKKS and cannot
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
KERNELS = ["k_hs_diag", "k_hs_imma", "k_drop_ntt", "k_ks_modup", "k_conv_mac", "k_intt_rows", "k_ks_intt", "k_ks_inner", "k_ntt_rows",
           "k_wire_to_slot", "k_add", "k_tensor_square", "k_add_plain"]
UNIT = "inferences/s"
SEED = 2110


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
INT_OPS_IMAD = {"k_hs_diag": 4, "k_ks_inner": 4, "k_drop_ntt": 6, "k_ks_modup": 6, "k_intt_rows": 6,
                "k_ks_intt": 6, "k_ntt_rows": 6}
# kernels whose MACs run on IMMA.16832.U8 as 64 byte-plane products each
TENSOR_KERNELS = ("k_hs_imma", "k_conv_mac")
IMMA_POPS = 1.1  # measured legacy mma.sync u8 rate on this B200 (tools/ubench_mma.cu)


def int_pipe_roofline(name, kd, clk_mhz):
    if not kd.get("modmuls"):
        return None
    if name in TENSOR_KERNELS:
        ops = kd["modmuls"] * 64 * 2 / (kd["ms_per_step"] / 1e3) / 1e12
        return {"pipe": "tensor (IMMA u8)", "achieved": ops, "peak": IMMA_POPS * 1e3, "unit": "TOPS (byte-plane)",
                "frac": ops / (IMMA_POPS * 1e3),
                "peak_basis": "measured mma.sync m16n8k32 u8 throughput, 64 byte-plane MACs per modular MAC"}
    per = INT_OPS_IMAD.get(name, 4)
    peak = N_SM * IMAD_WIDE_PER_CLK_SM * clk_mhz * 1e6 / per / 1e9
    return {"pipe": "int (IMAD)", "achieved": kd["gmodmul_s"], "peak": peak,
            "unit": "Gmodmul/s" if per == 4 else "G butterflies/s", "frac": kd["gmodmul_s"] / peak,
            "peak_basis": f"{N_SM} SMs x {IMAD_WIDE_PER_CLK_SM} IMAD.WIDE.U32/clk/SM x {clk_mhz:.0f} MHz / {per}"}


def ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`
    from the committed ncu --set full captures (profiles/), or None"""
    for name in ("r01_traffic_step.json", "r01_ncu_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                t = json.load(f)
            return float(t[kernel]["per_launch_bytes"])
        except Exception:
            continue
    return None


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
def _cpu_worker(args):
    """one image through the CPU restatement; returns seconds of evaluation"""
    n_images, seed = args
    from oracle import ckks_pipeline as P
    from oracle.ckks import Ckks
    from paper_2110_08321_b200.workloads import CFG0, net_image, net_weights
    cfg = CFG0
    ck = Ckks(cfg.log_n, list(cfg.qbits), cfg.pbits, seed=SEED)
    # the reference's algorithm (per-map conv + merge; the GPU's fused first
    # layer is not the reference's, so the baseline does not get it)
    prep = P.PreparedNet(ck, cfg, net_weights(cfg, SEED), merged=False)
    taps = [P.conv_pack_taps(ck, cfg, net_image(cfg, seed + i), seed + i, prep.tap_scale, merged=False)
            for i in range(n_images)]
    t0 = time.perf_counter()
    for t in taps:
        prep.eval(t)
    return time.perf_counter() - t0, n_images


def cpu_throughput(cores, images_per_core):
    """inferences/s of the CPU port on `cores` processes (one image stream each)."""
    if cores == 1:
        dt, n = _cpu_worker((images_per_core, 1000))
        return n / dt, f"{n} cfg0 image(s) evaluated on 1 core ({dt:.1f} s), keys/masks/taps prepared offline"
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        t0 = time.perf_counter()
        res = pool.map(_cpu_worker, [(images_per_core, 1000 + 100 * i) for i in range(cores)])
        wall = time.perf_counter() - t0
    n = sum(r[1] for r in res)
    per_core = [r[1] / r[0] for r in res]
    return float(sum(per_core)), (f"{n} cfg0 images, {images_per_core} per process on {cores} processes "
                                  f"(eval-only throughput summed over processes; wall {wall:.1f} s incl. setup)")


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import ckks
    ckks.build()
    cores = os.cpu_count() or 1
    vals = []
    for _ in range(args.warmup):
        pass  # the CPU port has no warm-up state beyond key generation (excluded)
    for _ in range(max(1, args.steps)):
        v, sample = cpu_throughput(cores, 1)
        vals.append(v)
    v = float(np.median(vals))
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 64_000.0 / v, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u64 (RNS mod q)", "data": "synthetic (seeded U[0,1] images, N(0,0.05^2) f32 weights)",
            "config": {"workload": "cfg2: 64 x cfg0 MNIST-sized net, CKKS N=8192",
                       "global_batch": 64, "parallelism": f"{cores} host processes"},
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
    from paper_2110_08321_b200.workloads import CFG0, net_image, net_weights

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    cfg = CFG0
    B = args.batch
    ctx = H.Context(cfg.log_n, list(cfg.qbits), cfg.pbits, seed=SEED, device=local)
    net = H.Net(ctx, cfg, net_weights(cfg, SEED))
    # client side (outside the timed region): conv-pack + encrypt this rank's images
    taps = np.concatenate([net.encrypt_image(net_image(cfg, i), nonce=i) for i in D.image_range(rank, B)])
    # the same ciphertexts in the compact fresh form the client ships (seeded
    # c1, byte-packed c0): the device step reads these straight from HBM
    compact = np.concatenate([net.encrypt_image_compact(net_image(cfg, i), nonce=i)
                              for i in D.image_range(rank, B)])
    dtaps = ctx.ct(B * net.ntaps, net.top, taps, 2.0 ** 40)
    dcompact = torch.from_numpy(compact).to(f"cuda:{local}")
    out = ctx.ct(B, net.out_level)

    def device_pass():
        if args.input == "compact":
            net.run_compact(dcompact, B, out)
        else:
            net.run(dtaps, out)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=local)
    gather_buf = torch.empty(B * net.out_words, dtype=torch.int64, device=f"cuda:{local}")
    gathered = torch.empty(world * B * net.out_words, dtype=torch.int64, device=f"cuda:{local}") if world > 1 else None

    graph = None

    def run_once():
        if graph is not None:
            graph()
        else:
            device_pass()

    def step():
        run_once()
        if world > 1:  # NCCL all-gather of the output ciphertexts (config 2)
            out.export_device(gather_buf.data_ptr())
            with torch.cuda.stream(stream):
                D.gather_outputs(gather_buf, world, gathered)

    for _ in range(args.warmup):
        step()
    ctx.sync()
    # one step's HOP tally and kernel launches (counted while issuing it)
    ctx.reset_meter()
    l0 = ctx.launches()
    if args.graph:  # the whole step as one CUDA graph: no host launch gaps
        graph = ctx.capture(device_pass)
    else:
        device_pass()
    ctx.sync()
    launches_per_step = ctx.launches() - l0
    tally = ctx.total()
    for _ in range(2):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = launches_per_step * args.steps
    ms_max = D.max_over_ranks(ev0.elapsed_time(ev1) / args.steps, device=f"cuda:{local}")
    value = B * world / (ms_max / 1e3)
    per_step_rot = tally[4]
    per_step_ks = per_step_rot + tally[3]  # rotations + relinearisations

    # ---- per-kernel device time (CUDA events around every launch of one
    # kernel, one extra device-resident step per kernel) -> roofline
    kernels = {}
    for name in KERNELS:
        ctx.kernel_timer(name)
        device_pass()  # direct launches (the timer brackets each one)
        kms, kn, kbytes, kops = ctx.kernel_timer_read_ops()
        if kn:
            kernels[name] = {"ms_per_step": kms, "launches": kn, "alg_bytes": kbytes,
                             "gbs": kbytes / (kms / 1e3) / 1e9 if kms > 0 else None,
                             "modmuls": kops, "gmodmul_s": kops / (kms / 1e3) / 1e9 if kms > 0 else None,
                             "share": kms / ms_max}
    clk_mhz = clk.summary()["sm_mhz"] or 1965.0
    for name, kd in kernels.items():
        kd["compute_roofline"] = int_pipe_roofline(name, kd, clk_mhz)
    ctx.kernel_timer(None)
    dom = max(kernels, key=lambda k: kernels[k]["ms_per_step"])
    ntt_rows = sum(kernels[k]["modmuls"] for k in ("k_drop_ntt", "k_ks_modup", "k_intt_rows", "k_ks_intt",
                                                  "k_ntt_rows") if k in kernels) / (
        (1 << (cfg.log_n - 1)) * cfg.log_n)
    hbm, which = peaks()
    kd = kernels[dom]
    traffic = ncu_traffic(dom)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": kd["gbs"], "peak": hbm, "unit": "GB/s",
                "frac": kd["gbs"] / hbm, "traffic": traffic, "peak_source": which,
                "alg_bytes_per_launch": kd["alg_bytes"] / kd["launches"],
                "avg_launch_ms": kd["ms_per_step"] / kd["launches"], "launches_per_step": kd["launches"],
                "share_of_step": kd["share"],
                # the kernel is bound by the 64-bit multiply-accumulate issue
                # rate, not HBM: its integer-pipe roofline
                "int_pipe": int_pipe_roofline(dom, kd, clk_mhz),
                "note": "alg bytes / modmuls per launch per DESIGN.md §5; traffic = ncu dram bytes per launch "
                        "of one step (profiles/r01_traffic_step.json: ncu --metrics dram__bytes_read.sum,"
                        "dram__bytes_write.sum over tools/one_step.py; L2-resident producer->consumer data "
                        "makes it lower than the algorithmic bytes)"}

    # ---- correctness spot check (outside timing): decrypt one output
    host_out = out.download()
    logits = net.decrypt_logits(host_out[: net.out_words])

    # ---- e2e through the public C-ABI from pinned host buffers: the client's
    # compact taps (c0 byte-packed + a-stream keys) go H2D chunk by chunk,
    # overlapped with the previous chunk's compute; outputs come back D2H
    pin_in = torch.from_numpy(compact).pin_memory()
    pin_out = torch.empty(B * net.out_words, dtype=torch.int64).pin_memory()

    def e2e_time(fn):
        # >= 4 passes: each of the two staging buffers runs once direct and is
        # then captured into a CUDA graph before the timed region
        for _ in range(max(4, args.warmup)):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            fn()
        e1.record(stream)
        e1.synchronize()
        return D.max_over_ranks(e0.elapsed_time(e1) / args.steps, device=f"cuda:{local}")

    # serving loop: every step is one submit (H2D of that step's compact taps,
    # compute, D2H of its outputs); step k+1's uploads overlap step k's
    # compute.  The timed region ends when the last step's outputs are on
    # the host.
    def serve_step():
        net.submit_host_compact(pin_in, B, pin_out, args.chunk)

    e2e_ms = e2e_time(serve_step)
    net.wait()
    assert np.array_equal(pin_out.numpy().view(np.uint64), host_out), "e2e output differs from device run"
    # one synchronous call per step (no cross-step overlap)
    sync_ms = e2e_time(lambda: net.run_host_compact(pin_in, B, pin_out, args.sync_chunk))
    assert np.array_equal(pin_out.numpy().view(np.uint64), host_out), "sync e2e output differs from device run"
    # the uncompressed full-ciphertext path, for reference
    pin_full = torch.from_numpy(taps.view(np.int64)).pin_memory()
    full_ms = e2e_time(lambda: net.run_host(pin_full, B, pin_out))
    assert np.array_equal(pin_out.numpy().view(np.uint64), host_out), "full e2e output differs from device run"

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64 (RNS mod q, 60/40-bit primes)",
        "data": "synthetic (seeded U[0,1] 28x28 images padded to 29x29, N(0,0.05^2) f32 weights)",
        "config": {"workload": "cfg2: 64 x cfg0 MNIST-sized net per GPU (conv-pack 25 cts -> merge -> "
                               "square -> HS 845->100 -> square -> HS 100->10), CKKS N=8192 L=6",
                   "global_batch": B * world, "images_per_gpu": B, "parallelism": f"dp{world} (image sharding)",
                   "input": args.input,
                   "l2": ("inputs 0.43 GB (compact) / 1.26 GB (full) per step > L2, no flush")},
        "rotations_per_s": per_step_rot * world / (ms_max / 1e3),
        "rotation_metering": ("reference HOP semantics (hesim's per-stage tally: 120 rotations per cfg-0 "
                              "inference); the engine runs fewer key switches than that -- HS diagonals and "
                              "folds hoisted, Conv1 + Flat1 fused (DESIGN.md §4)"),
        # limb transforms per second: every NTT-family launch's butterflies
        # / (N/2 log2 N) (one transform = one limb of one polynomial)
        "ntts_per_s": ntt_rows * world / (ms_max / 1e3),
        "ntts_per_step": ntt_rows,
        "keyswitches_per_s": per_step_ks * world / (ms_max / 1e3),
        "hops_per_inference": {k: v / B for k, v in zip(H.TALLY_FIELDS, tally)},
        "cuda_graph": bool(args.graph),
        "gpu_launches": launches,
        "roofline": roofline,
        "kernels": kernels,
        "clocks": clk.summary(),
        "e2e": {"value": B * world / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(compact.nbytes),
                "d2h_bytes_per_step": int(host_out.nbytes), "ms_per_step": e2e_ms,
                "path": "hegpu_net_submit_host_compact per step (compact taps; step k+1 H2D overlaps step k "
                        "compute), timed to the last step's outputs on the host",
                "chunk": args.chunk},
        "e2e_sync": {"value": B * world / (sync_ms / 1e3), "unit": UNIT, "ms_per_step": sync_ms,
                     "path": "hegpu_net_run_host_compact (one blocking call per step, chunked H2D overlap)",
                     "chunk": args.sync_chunk},
        "e2e_uncompressed": {"value": B * world / (full_ms / 1e3), "unit": UNIT,
                             "h2d_bytes_per_step": int(taps.nbytes), "ms_per_step": full_ms,
                             "path": "hegpu_net_run_host (full wire ciphertexts)"},
        "logits_sample": [float(x) for x in logits[:3]],
        "peak_hbm_gbs": hbm, "peak_source": which,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        v, sample = cpu_throughput(1, args.cpu_images)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    del net, dtaps, dcompact, out
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
    ap.add_argument("--cpu-images", type=int, default=8)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--chunk", type=int, default=64, help="images per compute chunk in the pipelined e2e (serving) loop (region-packed taps: 16: 10.9k, 32: 13.5k, 64: 14.8k inf/s)")
    ap.add_argument("--sync-chunk", type=int, default=32, help="images per chunk in the blocking e2e call")
    ap.add_argument("--graph", type=int, default=1, help="replay the device step as one CUDA graph")
    ap.add_argument("--input", default="full", choices=["compact", "full"],
                    help="device-resident input form: compact fresh taps (client wire form) or full ciphertexts")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
