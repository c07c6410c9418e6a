"""Print the TC kernel's per-tile pipeline timeline of CTA 0 (debug aid)."""
import os
import sys

os.environ["RANC_DEBUG_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_16208_b200 import Simulator  # noqa: E402
from workloads.gen import config3  # noqa: E402

net, inp = config3(S=int(sys.argv[1]) if len(sys.argv) > 1 else 10000)
sim = Simulator(net)
sim.load_inputs(inp)
sim.run(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
