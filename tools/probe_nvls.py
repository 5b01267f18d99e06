"""Probe (not product): multicast / NVLS availability on the GPU box at world size 1."""
import os, sys, torch, ctypes
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29531")
print("torch", torch.__version__, "gpus", torch.cuda.device_count())
from cuda.bindings import driver as drv
drv.cuInit(0)
err, dev = drv.cuDeviceGet(0)
for name in ["CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"]:
    a = getattr(drv.CUdevice_attribute, name, None)
    print(name, drv.cuDeviceGetAttribute(a, dev) if a is not None else "n/a")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
try:
    import torch.distributed._symmetric_memory as symm
    t = symm.empty(1 << 20, dtype=torch.int64, device="cuda:0")
    h = symm.rendezvous(t, dist.group.WORLD)
    print("symm ok; multicast_ptr", getattr(h, "multicast_ptr", None), "buffer_ptrs", getattr(h, "buffer_ptrs", None))
except Exception as e:
    print("symm failed:", type(e).__name__, e)
dist.destroy_process_group()
