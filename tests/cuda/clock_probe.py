"""Probe: SM clock (NVML, sampled every 20 ms) while the 12-layer cfg2
forward runs back to back for ~3 s, and the per-step time over that window.
Tells whether the tensor-heavy step runs at the max SM clock or power-caps."""
import ctypes as C
import os
import sys
import threading
import time

import numpy as np
import pynvml
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2508_01506_b200 import abi  # noqa: E402
from paper_2508_01506_b200.model import layer_descs, random_layer  # noqa: E402

L = abi.lib()
rng = np.random.default_rng(1234)
layers = [random_layer(768, 3072, 12, 12, 32, 384, 384, rng) for _ in range(12)]
descs = layer_descs(layers)
packs = []
for i in range(12):
    p = C.c_void_p()
    abi.check(L.fsvd_layer_pack_create(C.byref(descs[i]), abi.BF16, 0, C.byref(p)))
    packs.append(p)
parr = (C.c_void_p * 12)(*[p.value for p in packs])
B, M = 32, 512
wsb = C.c_size_t()
abi.check(L.fsvd_workspace_bytes_ln(parr, 12, B, M, abi.MODE_FLASH_V2, 0, C.byref(wsb)))
work = torch.empty(wsb.value, dtype=torch.uint8, device="cuda")
x = torch.randn((B, M, 768), device="cuda").to(torch.bfloat16)
out = torch.empty_like(x)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def fwd():
    abi.check(L.fsvd_model_fwd(parr, 12, abi.MODE_FLASH_V2, 0, B, M, C.c_void_p(x.data_ptr()),
                               C.c_void_p(out.data_ptr()), C.c_void_p(work.data_ptr()), wsb.value, sp))


pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples, stop = [], [False]


def sampler():
    while not stop[0]:
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
        time.sleep(0.02)


for _ in range(5):
    fwd()
torch.cuda.synchronize()
th = threading.Thread(target=sampler)
th.start()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 1200
a.record()
for _ in range(n):
    fwd()
b.record()
torch.cuda.synchronize()
stop[0] = True
th.join()
clk = np.array([s[0] for s in samples])
pw = np.array([s[1] for s in samples])
print(f"{n} back-to-back forwards: {a.elapsed_time(b) / n:.4f} ms/step; SM clock median {np.median(clk):.0f} "
      f"MHz (min {clk.min()}, max {clk.max()}), power median {np.median(pw):.0f} W max {pw.max():.0f} W, "
      f"throttle reasons seen {sorted(set(s[2] for s in samples))}, {len(samples)} samples")
