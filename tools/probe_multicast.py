"""Probe NVLS multicast support on the GPU box (driver attribute, torch
symmetric memory with a world of 1)."""
import ctypes
import os

import torch
import torch.distributed as dist

cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
v = ctypes.c_int(0)
r = cu.cuDeviceGetAttribute(ctypes.byref(v), 132, 0)
print("cuDeviceGetAttribute(MULTICAST_SUPPORTED) ->", r, v.value, flush=True)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29555")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
import torch.distributed._symmetric_memory as symm_mem

try:
    t = symm_mem.empty(1 << 20, dtype=torch.bfloat16, device="cuda:0")
    h = symm_mem.rendezvous(t, group=dist.group.WORLD)
    print("symm_mem ok: multicast_ptr =", hex(h.multicast_ptr), "buffer_ptrs", [hex(p) for p in h.buffer_ptrs],
          "t.data_ptr", hex(t.data_ptr()), flush=True)
except Exception as e:  # noqa: BLE001
    print("symm_mem failed:", type(e).__name__, e, flush=True)
dist.destroy_process_group()
