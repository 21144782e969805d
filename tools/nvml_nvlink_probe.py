"""Which NVLink counters does this driver expose?  NVML field values per
(field, scope) with their return codes, plus nvidia-smi's NVLink counters."""
import json
import subprocess

import pynvml

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
fields = {"COUNT_XMIT_BYTES": 202, "COUNT_RCV_BYTES": 204, "THROUGHPUT_DATA_TX": 138,
          "THROUGHPUT_DATA_RX": 139, "THROUGHPUT_RAW_TX": 140, "THROUGHPUT_RAW_RX": 141}
out = {}
for name, fid in fields.items():
    for scope in (0xFFFFFFFF, 0, 1, 17):
        try:
            v = pynvml.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            out[f"{name}/scope{scope:#x}"] = {"ret": int(v.nvmlReturn), "value": int(v.value.ullVal)}
        except pynvml.NVMLError as e:
            out[f"{name}/scope{scope:#x}"] = {"error": str(e)}
links = {}
for l in range(18):
    try:
        links[l] = int(pynvml.nvmlDeviceGetNvLinkState(h, l))
    except pynvml.NVMLError as e:
        links[l] = str(e)
out["link_state"] = links
for args in (["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], ["nvidia-smi", "nvlink", "-s", "-i", "0"]):
    r = subprocess.run(args, capture_output=True, text=True)
    out[" ".join(args)] = (r.stdout + r.stderr)[-1500:]
print(json.dumps(out, indent=1))
