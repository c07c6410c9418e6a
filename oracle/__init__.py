"""Serial CPU oracle of the RANC tick -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  It shares no code with the CUDA
product path (paper_2404_16208_b200/)."""
