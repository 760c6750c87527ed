"""Microbenchmark of the NVSwitch-multicast PS kernels vs NCCL, G ranks.
    torchrun --nproc-per-node G scripts/nvls_bench.py > gpurun_out/nvls_bench_gG.json
Per flat-buffer size (fp32 elements over all shards): the fused kernel
(multicast reduce + SGD + multicast bf16 store), its two halves alone, and
NCCL reduce-scatter (fp32) + all-gather (bf16) of the same buffers; CUDA events,
20 back-to-back launches, max over ranks."""
import ctypes
import json
import os
import sys

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1709_06622_b200 import device  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import nvlink_counters  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
L = device.lib()
vp = ctypes.c_void_p
L.tcb_ps_nvls_update.argtypes = [vp, vp, vp, vp, vp, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_float,
                                 ctypes.c_float, ctypes.c_float, ctypes.c_float, vp]
L.tcb_nvls_probe.argtypes = [ctypes.c_int, vp, vp, vp, vp, ctypes.c_size_t, ctypes.c_size_t, vp]


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    t = torch.tensor([s.elapsed_time(e) / reps], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


out = {"world": world, "device": torch.cuda.get_device_name(), "rows": []}
for n in (1 << 22, 1 << 24, 25_559_040):
    n = (n + 4 * world - 1) // (4 * world) * (4 * world)
    shard = n // world
    g = symm.empty(n, dtype=torch.float32, device="cuda")
    hg = symm.rendezvous(g, dist.group.WORLD.group_name)
    wc = symm.empty(n, dtype=torch.bfloat16, device="cuda")
    hw = symm.rendezvous(wc, dist.group.WORLD.group_name)
    gmc = hg.multicast_ptr + (g.data_ptr() - hg.buffer_ptrs[rank])
    wmc = hw.multicast_ptr + (wc.data_ptr() - hw.buffer_ptrs[rank])
    g.uniform_()
    w = torch.randn(n, device="cuda")
    v = torch.zeros(n, device="cuda")
    st = vp(torch.cuda.current_stream().cuda_stream)
    o = rank * shard
    fused_fn = lambda: L.tcb_ps_nvls_update(vp(gmc), vp(g.data_ptr()), vp(w.data_ptr()), vp(v.data_ptr()),  # noqa: E731
                                            vp(wmc), o, shard, 0.0, 0.9, 0.0, 1.0 / world, st)
    fused = timeit(fused_fn)
    # NVLink hardware byte counters of this GPU over 20 fused launches
    torch.cuda.synchronize()
    dist.barrier()
    c0 = nvlink_counters.read(int(os.environ["LOCAL_RANK"]))
    for _ in range(20):
        fused_fn()
    torch.cuda.synchronize()
    c1 = nvlink_counters.read(int(os.environ["LOCAL_RANK"]))
    dist.barrier()
    cnt = nvlink_counters.delta(c0, c1)
    red = timeit(lambda: L.tcb_nvls_probe(1, vp(gmc), vp(g.data_ptr()), vp(w.data_ptr()), vp(wmc), o, shard, st))
    sto = timeit(lambda: L.tcb_nvls_probe(2, vp(gmc), vp(g.data_ptr()), vp(w.data_ptr()), vp(wmc), o, shard, st))
    gl = torch.empty(n, device="cuda")
    wl = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    rs = timeit(lambda: dist.reduce_scatter_tensor(gl[o:o + shard], gl))
    ag = timeit(lambda: dist.all_gather_into_tensor(wl, wl[o:o + shard]))
    torch.cuda.synchronize()
    dist.barrier()
    r0 = nvlink_counters.read(int(os.environ["LOCAL_RANK"]))
    for _ in range(20):
        dist.reduce_scatter_tensor(gl[o:o + shard], gl)
        dist.all_gather_into_tensor(wl, wl[o:o + shard])
    torch.cuda.synchronize()
    r1 = nvlink_counters.read(int(os.environ["LOCAL_RANK"]))
    dist.barrier()
    rcnt = nvlink_counters.delta(r0, r1)
    row = {"flat_fp32_MB": round(n * 4 / 1e6, 2), "shard_elems": shard,
           "fused_ms": round(fused, 4), "reduce_only_ms": round(red, 4), "store_only_ms": round(sto, 4),
           "nccl_rs_ms": round(rs, 4), "nccl_ag_bf16_ms": round(ag, 4),
           "reduce_GBps_per_gpu": round(shard * 4 / red / 1e6, 1),
           "nccl_rs_busbw_GBps": round(n * 4 * (world - 1) / world / rs / 1e6, 1),
           "nvlink_counters_rank0_fused_x20": cnt,
           "nvlink_counters_rank0_fused_per_launch_GB": (
               {k: round(v / 20 / 1e9, 4) for k, v in cnt.items()} if cnt else None),
           "nvlink_counters_rank0_nccl_rs_ag_x20": rcnt,
           "nvlink_counters_rank0_nccl_per_step_GB": (
               {k: round(v / 20 / 1e9, 4) for k, v in rcnt.items()} if rcnt else None),
           # per GPU and launch: NVLS reads every GPU's whole fp32 buffer through the switch
           # (own shard included) and multicasts the bf16 shard once; RS + AG move the
           # other ranks' (G-1)/G of the fp32 buffer out and the bf16 shard to G-1 peers
           "model_egress_GB_fused": round((n * 4 + shard * 2) / 1e9, 4),
           "model_egress_GB_rs_ag": round((shard * 4 * (world - 1) + shard * 2 * (world - 1)) / 1e9, 4)}
    out["rows"].append(row)
    del g, wc, hg, hw
if rank == 0:
    print(json.dumps(out, indent=1))
dist.barrier()
dist.destroy_process_group()
