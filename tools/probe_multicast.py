"""Probe NVLS multicast support on this box (f4 multimem epilogue): torch
SymmetricMemory on a 1-rank group; prints has_multicast_support and whether a
multicast pointer is handed out."""
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
print("has_multicast_support:", torch._C._distributed_c10d._SymmetricMemory.has_multicast_support(
    symm_mem.DeviceType.CUDA, 0))
try:
    t = symm_mem.empty((1024, 128), dtype=torch.float32, device="cuda")
    h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
    print("multicast_ptr:", h.multicast_ptr, "buffer_ptrs:", h.buffer_ptrs)
except Exception as e:  # noqa: BLE001
    print("symm_mem error:", repr(e)[:500])
dist.destroy_process_group()
