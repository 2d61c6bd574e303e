import time, pynvml
pynvml.nvmlInit(); h=pynvml.nvmlDeviceGetHandleByIndex(0)
for f in ("clock", "reasons", "max"):
    t=time.perf_counter()
    for _ in range(20):
        if f=="clock": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        elif f=="reasons": pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        else: pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
    print(f, (time.perf_counter()-t)/20*1e3, "ms")
