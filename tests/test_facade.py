"""Host-side unit tests of the C++ graphqc facade (tests/facade_test.cpp): the
reference's graph / metrics / sweep test cases that need no device."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2305_14641_b200")
SRC = os.path.join(ROOT, "tests", "facade_test.cpp")
BIN = os.path.join(ROOT, "tests", "_build", "facade_test")


def test_facade_host_units():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    subprocess.check_call(["g++", "-O1", "-std=c++20", "-ffp-contract=off", "-I", os.path.join(PKG, "host", "include"),
                           "-I", os.path.join(ROOT, "include"), "-o", BIN, SRC, "-L", PKG, "-lgraphqc", "-lgqc",
                           f"-Wl,-rpath,{PKG}"])
    r = subprocess.run([BIN, os.path.join(ROOT, "tests", "golden")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "facade host tests passed" in r.stdout
    # the conflicting duplicate edge in the round-trip case is reported like graph.cpp:48-51
    assert "warning: duplicate edge 3 17 keeps weight 0.75, ignoring 0.5" in r.stderr
