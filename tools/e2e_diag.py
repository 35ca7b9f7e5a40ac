"""Where does the pipelined e2e step go?  Times (device events) the serving
loop, the pure H2D of one step's compact taps, and per-kernel totals inside
the loop.  python tools/e2e_diag.py"""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2110_08321_b200 import hegpu as H
from paper_2110_08321_b200.workloads import CFG0, net_image, net_weights

B = 64
cfg = CFG0
ctx = H.Context(cfg.log_n, list(cfg.qbits), cfg.pbits, seed=2110)
net = H.Net(ctx, cfg, net_weights(cfg, 2110))
compact = np.concatenate([net.encrypt_image_compact(net_image(cfg, i), nonce=i) for i in range(B)])
pin_in = torch.from_numpy(compact).pin_memory()
pin_out = torch.empty(B * net.out_words, dtype=torch.int64).pin_memory()
stream = torch.cuda.ExternalStream(ctx.stream_ptr())
chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 64

def timed(fn, k=6):
    for _ in range(2):
        fn()
    net.wait(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        fn()
    e1.record(stream); e1.synchronize(); net.wait()
    return e0.elapsed_time(e1) / k

print("serve step ms", timed(lambda: net.submit_host_compact(pin_in, B, pin_out, chunk)))
d = torch.empty(compact.nbytes, dtype=torch.uint8, device="cuda")
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record(); [d.copy_(pin_in, non_blocking=True) for _ in range(5)]; t1.record(); t1.synchronize()
print("pure H2D ms", t0.elapsed_time(t1) / 5)
for k in ["k_expand_compact", "k_conv_mac", "k_hs_diag", "k_drop_ntt", "k_ks_modup", "k_intt_rows", "k_ks_intt", "k_ks_inner"]:
    ctx.kernel_timer(k)
    net.run_host_compact(pin_in, B, pin_out, chunk)
    ms, n, b = ctx.kernel_timer_read()
    print(k, round(ms, 3), n)
ctx.kernel_timer(None)

# H2D bandwidth alone vs while the network runs on the engine stream
dcompact = torch.from_numpy(compact).cuda()
out = ctx.ct(B, net.out_level)
side = torch.cuda.Stream()
def h2d_ms(concurrent):
    torch.cuda.synchronize(); net.wait()
    if concurrent:
        for _ in range(6):
            net.run_compact(dcompact, B, out)
    with torch.cuda.stream(side):
        a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
        a0.record(side)
        for _ in range(4):
            d.copy_(pin_in, non_blocking=True)
        a1.record(side)
    a1.synchronize()
    ctx.sync()
    return a0.elapsed_time(a1) / 4
print("H2D ms alone", h2d_ms(False), "during compute", h2d_ms(True))

# host-side enqueue time per serving pass (GPU busy or not)
net.wait()
t0 = time.perf_counter()
for _ in range(5):
    net.submit_host_compact(pin_in, B, pin_out, chunk)
t1 = time.perf_counter()
net.wait()
t2 = time.perf_counter()
print("host enqueue ms/pass", (t1 - t0) / 5 * 1e3, "wall ms/pass", (t2 - t0) / 5 * 1e3)
t0 = time.perf_counter()
for _ in range(5):
    net.run_compact(dcompact, B, out)
t1 = time.perf_counter()
ctx.sync()
t2 = time.perf_counter()
print("host enqueue ms/run_compact", (t1 - t0) / 5 * 1e3, "wall", (t2 - t0) / 5 * 1e3)

# network compute time with and without a concurrent H2D stream
def compute_ms(concurrent, k=5):
    torch.cuda.synchronize(); ctx.sync()
    eng = torch.cuda.ExternalStream(ctx.stream_ptr())
    if concurrent:
        with torch.cuda.stream(side):
            for _ in range(8):
                d.copy_(pin_in, non_blocking=True)
    c0e = torch.cuda.Event(enable_timing=True); c1e = torch.cuda.Event(enable_timing=True)
    c0e.record(eng)
    for _ in range(k):
        net.run_compact(dcompact, B, out)
    c1e.record(eng)
    c1e.synchronize()
    torch.cuda.synchronize()
    return c0e.elapsed_time(c1e) / k
print("run_compact ms alone", compute_ms(False), "with concurrent H2D", compute_ms(True))
