"""Probe (one GPU): multicast / NVLS support and torch symmetric memory at world size 1 — whether
a fused wgrad-GEMM + multimem all-reduce can even be exercised on a 1-GPU lease."""
import os

import torch
import torch.distributed as dist

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
print("torch", torch.__version__, torch.cuda.get_device_name(0))
try:
    from cuda.bindings import driver as cu   # cuda-python
    cu.cuInit(0)
    err, dev = cu.cuDeviceGet(0)
    err, mc = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
    print("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED:", mc, err)
except Exception as e:  # noqa: BLE001
    print("cuda-python probe failed:", type(e).__name__, e)
torch.cuda.set_device(0)
for backend in ("nccl",):
    try:
        dist.init_process_group(backend, rank=0, world_size=1, device_id=torch.device("cuda", 0))
        import torch.distributed._symmetric_memory as symm_mem
        t = symm_mem.empty(1024, dtype=torch.float32, device="cuda")
        h = symm_mem.rendezvous(t, dist.group.WORLD)
        print("symm_mem rendezvous ok: world", h.world_size, "buffer_ptrs", [hex(p) for p in h.buffer_ptrs],
              "multicast_ptr", hex(h.multicast_ptr) if getattr(h, "multicast_ptr", 0) else h.multicast_ptr)
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        print(backend, "symm_mem failed:", type(e).__name__, str(e)[:300])
