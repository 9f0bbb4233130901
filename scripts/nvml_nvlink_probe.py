"""Which NVML NVLink throughput counters this box exposes (field values
NVLINK_THROUGHPUT_DATA_TX/RX, per link and aggregate)."""
import pynvml as nv

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
for fid in (nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX):
    for scope in (None, 0, 1, 0xFFFFFFFF):
        try:
            arg = [fid] if scope is None else [(fid, scope)]
            v = nv.nvmlDeviceGetFieldValues(h, arg)[0]
            print(fid, scope, "ret", v.nvmlReturn, "type", v.valueType, "ull", v.value.ullVal)
        except Exception as e:
            print(fid, scope, "exc", e)
try:
    print("links active:", sum(1 for l in range(18)
                               if nv.nvmlDeviceGetNvLinkState(h, l) == nv.NVML_FEATURE_ENABLED))
except Exception as e:
    print("link state exc", e)
