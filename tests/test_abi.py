"""CPU tests of the C-ABI boundary: the library loads, exports every symbol
include/ranc.h declares, validates networks with located errors, and has no
CPU fallback."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2404_16208_b200 import _lib, build
    build.build()
    return _lib.load()


def header_functions():
    src = open(os.path.join(ROOT, "include", "ranc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ranc_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    fns = header_functions()
    assert len(fns) >= 19
    for f in fns:
        assert hasattr(lib, f), f
    from paper_2404_16208_b200 import _lib
    assert set(_lib.EXPORTS) == set(fns)


def test_so_is_sm100a():
    import subprocess
    from paper_2404_16208_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _net():
    from workloads.gen import config2
    net, _ = config2(S=1)
    return net


def expect(status, code, fragment, net_mut):
    from paper_2404_16208_b200 import RancError, Simulator
    net = _net()
    net_mut(net)
    with pytest.raises(RancError) as ei:
        Simulator(net)
    assert ei.value.code == code, str(ei.value)
    assert fragment in str(ei.value), str(ei.value)


def test_located_validation_errors(lib):
    def w(n): n.weight[2, 17, 1] = 300
    expect(None, "RANC_E_BITWIDTH", "core (2,0) neuron 17: weight[1]=300 exceeds weight_bits=9", w)

    def leak(n): n.leak[1, 3] = -1000
    expect(None, "RANC_E_BITWIDTH", "core (1,0) neuron 3: leak=-1000", leak)

    def off(n):
        n.dest_kind[4, 0] = 1
        n.dest_dx[4, 0] = 1
    expect(None, "RANC_E_OFFGRID", "core (4,0) neuron 0: route (dx=1,dy=0) leaves the 5x1 grid", off)

    def delay(n):
        n.dest_delay[0, 5] = 2
    expect(None, "RANC_E_RANGE", "dest_delay=2 not in [1,1]", delay)

    def delay0(n):
        n.dest_delay[0, 5] = 0          # G7: delay 0 is rejected
    expect(None, "RANC_E_RANGE", "dest_delay=0", delay0)

    def ty(n): n.axon_type[3, 9] = 4
    expect(None, "RANC_E_RANGE", "core (3,0) axon 9: axon_type=4 >= num_types=4", ty)

    def cls(n): n.out_class[4, 2] = 10
    expect(None, "RANC_E_RANGE", "out_class=10 >= num_classes=10", cls)

    def line(n): n.input_line[0, 0] = 784
    expect(None, "RANC_E_RANGE", "input_line=784", line)

    def mode(n): n.reset_mode[0, 0] = 2
    expect(None, "RANC_E_RANGE", "reset_mode=2", mode)

    def bits(n): n.potential_bits = 17
    expect(None, "RANC_E_CONFIG", "potential_bits=17", bits)

    def d16(n): n.max_delay = 16
    expect(None, "RANC_E_CONFIG", "max_delay=16", d16)


def test_padding_bits_rejected(lib):
    from workloads.gen import random_network
    from paper_2404_16208_b200 import RancError, Simulator
    net = random_network(1, 1, 1, 33, 4, 2, 2)
    net.crossbar[0, 1, 1] |= np.uint32(1 << 5)
    with pytest.raises(RancError) as ei:
        Simulator(net)
    assert ei.value.code == "RANC_E_RANGE" and "beyond axons" in str(ei.value)


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2404_16208_b200 import RancError, Simulator
    with pytest.raises(RancError) as ei:
        Simulator(_net())
    assert ei.value.code == "RANC_E_CUDA" and "no CPU fallback" in str(ei.value)


def test_null_args(lib):
    assert lib.ranc_run_ticks(None, 1) == 1
    assert lib.ranc_read_outputs(None, None, 0) == 1
    h = ctypes.c_void_p()
    assert lib.ranc_load_network(None, 0, ctypes.byref(h)) == 1
    assert b"NULL" in lib.ranc_last_error(None)
    lib.ranc_destroy(None)


def test_plain_c99_consumer(lib, tmp_path):
    """The header is plain C99: a consumer compiled with gcc -std=c99
    -pedantic -Werror and linked to libranc.so runs the host-only entry
    points (core-shard planner, located validation error, NULL arguments, no
    CPU fallback) -- tests/c/consumer.c."""
    import subprocess
    from paper_2404_16208_b200 import _lib
    exe = str(tmp_path / "consumer")
    libdir = os.path.dirname(_lib.LIB_PATH)
    cc = ["gcc", "-std=c99", "-pedantic", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "include"),
          os.path.join(ROOT, "tests", "c", "consumer.c"), "-o", exe, "-L" + libdir, "-l:libranc.so",
          "-Wl,-rpath," + libdir]
    r = subprocess.run(cc, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
