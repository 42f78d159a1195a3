"""Step time over a long graph-replay run, in windows, with nvidia-smi samples
(SM / memory clock, power) taken during the run.
  python tools/probes/steady_state.py [workload] [steps]"""
import json
import subprocess
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import WORKLOADS  # noqa: E402
from paper_2303_06182_b200.layer import LayerShape, MoeLayer, make_tokens, make_weights  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "lm"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 400
S, TD, HD, E, k, mode, C, _ = WORKLOADS[wl]
shape = LayerShape(TD, HD, E, k)
L = MoeLayer(shape, S, weights=make_weights(shape))
x = make_tokens(S, TD)
out = torch.empty_like(x)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(5):
        L.forward(x, out, graph=True, stream=s)
s.synchronize()
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,"
                            "clocks_event_reasons.active", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True).stdout.strip()
        samples.append((time.time(), r))
        time.sleep(0.05)


th = threading.Thread(target=sampler)
th.start()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
t0 = time.time()
with torch.cuda.stream(s):
    for i in range(K):
        ev[i].record(s)
        L.forward(x, out, graph=True, stream=s)
    ev[K].record(s)
s.synchronize()
stop.set()
th.join()
st = np.array([ev[i].elapsed_time(ev[i + 1]) for i in range(K)])
W = max(1, K // 8)
print(json.dumps({"workload": wl, "steps": K, "window_ms_mean": [round(float(st[i:i + W].mean()), 4) for i in range(0, K, W)],
                  "p50": float(np.median(st)), "min": float(st.min()), "max": float(st.max())}))
for t, r in samples[:: max(1, len(samples) // 12)]:
    print(f"{t - t0:6.2f}s  sm,mem MHz / W / C / reasons: {r}")
