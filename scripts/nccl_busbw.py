"""NVLink bus bandwidth of the PS collectives on this box: NCCL reduce-scatter
(fp32 sum) and all-gather (bf16) over message sizes up to the ResNet-50 / VGG-16
flat parameter buffers; busbw = S * (G - 1) / G / t (device-timed, max over
ranks). The peak RS/AG busbw is the denominator of the PS-aggregation roofline.

    torchrun --nproc-per-node G --master-addr 127.0.0.1 scripts/nccl_busbw.py > out.json
"""
import json
import os

import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    res = []
    for mb in (8, 32, 102, 256, 553, 1024):
        n = mb * 2**20 // 4 // (world * 64) * world * 64
        for op, dt in (("reduce_scatter", torch.float32), ("all_gather", torch.bfloat16)):
            full = torch.ones(n, dtype=dt, device="cuda")
            shard = torch.empty(n // world, dtype=dt, device="cuda")
            fn = (lambda: dist.reduce_scatter_tensor(shard, full)) if op == "reduce_scatter" else \
                 (lambda: dist.all_gather_into_tensor(full, shard))
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            dist.barrier()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 20
            s.record()
            for _ in range(reps):
                fn()
            e.record()
            e.synchronize()
            t = torch.tensor([s.elapsed_time(e) / reps], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            nbytes = n * full.element_size()
            res.append({"op": op, "bytes": nbytes, "ms": round(ms, 4),
                        "busbw_GBps": round(nbytes * (world - 1) / world / (ms / 1e3) / 1e9, 1)})
    if rank == 0:
        print(json.dumps({"gpus": world, "nccl": ".".join(map(str, torch.cuda.nccl.version())),
                          "results": res}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
