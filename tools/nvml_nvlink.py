"""Probe: NVML NVLink throughput field values (data/raw tx/rx, KiB) per GPU."""
import json, sys
import pynvml as N
N.nvmlInit()
out = {}
F = {"data_tx": 138, "data_rx": 139, "raw_tx": 140, "raw_rx": 141}
for i in range(N.nvmlDeviceGetCount()):
    h = N.nvmlDeviceGetHandleByIndex(i)
    vals = {}
    for name, fid in F.items():
        try:
            r = N.nvmlDeviceGetFieldValues(h, [fid])[0]
            vals[name] = (int(r.nvmlReturn), int(r.value.ullVal))
        except Exception as e:
            vals[name] = str(e)
    out[i] = vals
print(json.dumps(out))
