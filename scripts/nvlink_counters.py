"""NVLink hardware byte counters (NVML field values NVLINK_THROUGHPUT_DATA_TX /
RX, KiB, summed over all links of a GPU). Used around PS-step microbenchmarks
to report the bytes that actually crossed each GPU's NVLinks — a hardware
counter read, since the profiling guide rules out ncu on multi-rank runs."""
import pynvml

_FIELDS = None


def _init():
    global _FIELDS
    if _FIELDS is None:
        pynvml.nvmlInit()
        _FIELDS = (pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX,
                   pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX, pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX)


def read(gpu_index):
    """{data_tx, data_rx, raw_tx, raw_rx} in bytes (cumulative) for one GPU, or
    None when the counters are not readable."""
    try:
        _init()
        h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
        vals = pynvml.nvmlDeviceGetFieldValues(h, list(_FIELDS))
        out = {}
        for name, v in zip(("data_tx", "data_rx", "raw_tx", "raw_rx"), vals):
            if v.nvmlReturn != 0:
                return None
            out[name] = int(v.value.ullVal) * 1024
        return out
    except Exception:  # noqa: BLE001 — counters are optional evidence
        return None


def delta(before, after):
    if not before or not after:
        return None
    return {k: after[k] - before[k] for k in before}
