"""Probe: torch symmetric memory + NVLS multicast availability on this box.
    torchrun --nproc-per-node 2 scripts/nvls_probe.py"""
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

rank = int(os.environ["RANK"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl")
t = symm.empty(1 << 20, dtype=torch.float32, device="cuda")
h = symm.rendezvous(t, dist.group.WORLD.group_name)
attrs = {k: getattr(h, k) for k in dir(h) if not k.startswith("_")}
print(rank, "multicast_ptr", hex(h.multicast_ptr), "buffer_ptrs", [hex(p) for p in h.buffer_ptrs],
      "signal_pad_ptrs", [hex(p) for p in h.signal_pad_ptrs], "signal_pad_size", h.signal_pad_size,
      "attrs", sorted(attrs), flush=True)
dist.barrier()
dist.destroy_process_group()
