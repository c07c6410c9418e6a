"""us/tick of the streaming workload: per-tick launches vs one cooperative launch."""
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2404_16208_b200 import OPT_STREAM, Simulator  # noqa: E402
from workloads.gen import config3_stream  # noqa: E402

n_img = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
net, inp = config3_stream(n_img)
T = net.meta["T"]
for opt in (1, 2):
    sim = Simulator(net)
    sim.set_option(OPT_STREAM, opt)
    sim.load_inputs(inp)
    sim.run(T)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        sim.reset()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sim.run(T)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"stream opt {opt}: {T} ticks in {best * 1e3:.2f} ms = {best / T * 1e6:.2f} us/tick", flush=True)
    sim.close()
