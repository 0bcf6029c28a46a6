"""Drop-in proof: the reference's own release gate (proj/tests/acceptance.cpp,
criteria C1-C9) compiled unmodified and linked against the B200 engine through
integration/pslopt_search_b200.cpp, which replaces the reference's
src/search.cpp (run_search, neighborhood_scan, ... over the C ABI).
Built by `make -C oracle dropin` where /root/reference exists; the binary
travels with the repo snapshot to the GPU box."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(BIN), reason="acceptance_b200 not built")]


def run(crit, timeout):
    p = subprocess.run([BIN, str(crit)], capture_output=True, text=True, timeout=timeout)
    return p.returncode, p.stdout + p.stderr


# C1 incremental==brute, C2 exhaustive optima, C3 MF identity, C6 records
# identical across worker counts (L=4095, 1e6 NSE), C8 invariant suite, C9 format
# round trips -- all through the GPU run_search.
@pytest.mark.parametrize("crit", [1, 2, 3, 6, 8, 9])
def test_acceptance_criterion(crit):
    rc, out = run(crit, 900)
    assert rc == 0 and "PASS" in out, out


# C4 two-phase ablation ordering (30 runs of 1e7 NSE at L=1023) and C5 quality
# headline (10 runs) -- quality gates of the search itself, on the GPU.
@pytest.mark.parametrize("crit", [4, 5])
def test_acceptance_quality(crit):
    rc, out = run(crit, 1800)
    assert rc == 0 and "PASS" in out, out
