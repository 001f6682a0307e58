"""SM clock under a long bf16 GEMM loop, three readers side by side: NVML nvmlDeviceGetClockInfo,
NVML nvmlDeviceGetClock(CURRENT), and `nvidia-smi -lms 20` (what bench.py's ClockSampler can use)."""
import json
import statistics
import subprocess
import threading
import time

import pynvml
import torch

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByUUID("GPU-" + str(torch.cuda.get_device_properties(0).uuid))
rows = {"info": [], "current": [], "smi": []}
halt = threading.Event()


def poll():
    while not halt.is_set():
        rows["info"].append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        rows["current"].append(pynvml.nvmlDeviceGetClock(h, pynvml.NVML_CLOCK_SM, pynvml.NVML_CLOCK_ID_CURRENT))
        time.sleep(0.005)


smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-lms", "20"],
                       stdout=subprocess.PIPE, text=True)
a = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda")
for _ in range(20):
    a @ b
torch.cuda.synchronize()
th = threading.Thread(target=poll, daemon=True)
th.start()
t0 = time.perf_counter()
n = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.perf_counter() - t0 < 3.0:
    for _ in range(10):
        a @ b
    n += 10
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
halt.set()
th.join()
smi.terminate()
out = smi.communicate()[0]
rows["smi"] = [float(x) for x in out.split() if x.strip().replace(".", "").isdigit()]
ms = e0.elapsed_time(e1)
print(json.dumps({"tflops": 2 * 8192 ** 3 * n / ms / 1e9, "gemms": n,
                  **{k: {"n": len(v), "median": statistics.median(v) if v else None, "min": min(v) if v else None,
                         "max": max(v) if v else None} for k, v in rows.items()}}))
