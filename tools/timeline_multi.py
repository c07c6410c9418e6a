"""Per-item pipeline timeline of CTA 0 in the multi-tick (cooperative)
tensor-core launch (RANC_DEBUG_TIMELINE_MULTI): pipeline index k = tick *
items-per-CTA + item.  python tools/timeline_multi.py [vmm256|config2] [ticks]"""
import os
import sys

os.environ["RANC_DEBUG_TIMELINE_MULTI"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_16208_b200 import Simulator  # noqa: E402
from workloads import gen  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "vmm256"
net, inp = gen.config4("vmm256", S=1000) if wl == "vmm256" else gen.config2(S=1000)
sim = Simulator(net)
sim.set_option(3, 2)
sim.load_inputs(inp)
sim.run(int(sys.argv[2]) if len(sys.argv) > 2 else 40)
