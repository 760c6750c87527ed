"""Measured NVLink peak on this box (one process, all visible GPUs):
per-direction peer copy GPU0 -> GPU1 (copy engine, 1 GiB, best of 10) and
bidirectional, with the NVML NVLink byte counters read around the copies to
validate them. Writes profiles-ready JSON to stdout.
    python scripts/nvlink_peak.py > gpurun_out/nvlink_peak_g<N>.json"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import nvlink_counters  # noqa: E402

n = torch.cuda.device_count()
assert n >= 2, "needs 2 GPUs"
nbytes = 1 << 30
a = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")
b = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
a.fill_(1)
b.fill_(2)
b2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
a2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")


def best(fn, reps=10, dev=0):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        with torch.cuda.device(dev):
            s.record()
            fn()
            e.record()
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        ts.append(s.elapsed_time(e))
    return min(ts)


best(lambda: b.copy_(a, non_blocking=True))
c0 = nvlink_counters.read(0)
uni = best(lambda: b.copy_(a, non_blocking=True))
c1 = nvlink_counters.read(0)
s1 = torch.cuda.Stream(device=1)


def bidir():
    b.copy_(a, non_blocking=True)
    with torch.cuda.stream(s1):
        a2.copy_(b2, non_blocking=True)
    torch.cuda.current_stream(0).wait_stream(s1)


bi = best(bidir)
out = {"gpus": n, "device": torch.cuda.get_device_name(0), "bytes": nbytes,
       "peer_copy_GBps_per_direction": round(nbytes / uni / 1e6, 1),
       "peer_copy_bidirectional_GBps": round(2 * nbytes / bi / 1e6, 1),
       "method": "torch copy_ GPU0->GPU1 (cudaMemcpyPeerAsync, copy engine), best of 10, CUDA events",
       "nvml_counters_gpu0_over_10_unidir_copies": nvlink_counters.delta(c0, c1),
       "expected_tx_bytes": 10 * nbytes}
print(json.dumps(out, indent=1))
