"""Print the TC kernel's per-tile pipeline timeline of CTA 0 (debug aid).

  python tools/timeline.py [config3|config5|config5g|<bench workload>] [S] [ticks] [ring layout 0-3] [operand 0-2]
"""
import os
import sys

os.environ["RANC_DEBUG_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_16208_b200 import Simulator  # noqa: E402
from workloads import gen  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "config3"
S = int(sys.argv[2]) if len(sys.argv) > 2 else (64 if wl.startswith("config5") else 10000)
if wl == "config3":
    net, inp = gen.config3(S=S)
elif wl.startswith("config5"):
    net, inp = gen.config5(S=S, T=10, variant="global" if wl == "config5g" else "local")
else:   # any bench.py workload (its default sample count unless S > 0)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench  # noqa: E402
    builder, S0, _ = bench.WORKLOADS[wl]
    net, inp = builder(S if S > 0 else S0)
sim = Simulator(net)
sim.set_option(3, 2)
if len(sys.argv) > 4:
    sim.set_option(5, int(sys.argv[4]))
if len(sys.argv) > 5:
    sim.set_option(7, int(sys.argv[5]))   # RANC_OPT_OPERAND
sim.load_inputs(inp)
sim.run(int(sys.argv[3]) if len(sys.argv) > 3 else 3)
