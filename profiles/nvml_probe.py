"""How long do NVML clock / throttle-reason queries take (and do they stall a running solve)?"""
import time
import pynvml

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
for name, fn in (("clock", lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                 ("reasons", lambda: pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)),
                 ("maxclock", lambda: pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))):
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e3)
        time.sleep(0.02)
    print(f"{name:9s} ms: first {ts[0]:.2f}  median {sorted(ts)[15]:.3f}  max {max(ts):.2f}")
