"""Drop-in proof: the reference's own release gate (proj/tests/acceptance.cpp,
criteria C1-C9) compiled unmodified and linked against the B200 engine through
integration/pslopt_search_b200.cpp and integration/pslopt_sequence_b200.cpp,
which replace the reference's src/search.cpp and src/sequence.cpp.
Built by `make -C oracle dropin` where /root/reference exists; the binary
travels with the repo snapshot to the GPU box.

What each criterion exercises on the GPU (acceptance.cpp line numbers):
  C1 (:75-99)   SidelobeTable::build + evaluate_neighbor on the engine, checked
                against the reference's CPU oracle::brute_fitness (oracle.cpp)
  C3 (:150-169) build + fitness (serial device chain) + merit_factor
  C4, C5, C6    run_search (the device-resident walk)
  C8 (:283-382) build + apply_flip on the engine, run_search accounting
  C2 (:102-148) and C9 (:397-) call only the reference's own oracle.cpp / io.cpp
                (exhaustive search, text round trips): CPU reference code that
                stays in the link; they show the relinked library is complete,
                not that the engine is right.
"""
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


# C1 incremental==brute, C2 exhaustive optima (CPU oracle.cpp), C3 MF identity,
# C6 records identical across worker counts (L=4095, 1e6 NSE), C8 invariant
# suite, C9 format round trips (CPU io.cpp) -- see the module docstring.
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


CLI = os.path.join(ROOT, "oracle", "_ref", "pslopt_b200")

# docs/formats.md:31-55 (the reference's own golden record); elapsed masked
FORMATS_MD_RECORD = """pslopt-run v1
length: 16
seed: 3
alpha1: 4
alpha2: 13
ls-lmt: 2000
flip-lmt: 10
n-lmt: 16
workers: 1
max-nse: 400
max-seconds: none
init: none
solver-version: 0.1.0
nse: 401
elapsed-seconds: *
psl-best: 2
merit-factor: 4.571428571428571
solution-best: +-+-++--++-----+
events: 4
event: 17 * 3 1 improved-psl
event: 17 * 3 1 local-best-improved
event: 49 * 2 1 improved-psl
event: 49 * 2 1 local-best-improved
"""


def _mask(text):
    out = []
    for line in text.splitlines():
        if line.startswith("elapsed-seconds:"):
            line = "elapsed-seconds: *"
        elif line.startswith("event:"):
            f = line.split()
            f[2] = "*"
            line = " ".join(f)
        out.append(line)
    return "\n".join(out) + "\n"


@pytest.mark.skipif(not os.path.exists(CLI), reason="pslopt_b200 not built")
def test_cli_solve_writes_reference_record(tmp_path):
    out, best, log = tmp_path / "rec.txt", tmp_path / "best.txt", tmp_path / "log.csv"
    p = subprocess.run([CLI, "solve", "-L", "16", "--seed", "3", "--n-lmt", "16", "--max-nse", "400",
                        "--out", str(out), "--best", str(best), "--log", str(log)],
                       capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stderr
    assert p.stdout.startswith("PSL=2 NSE=401 MF=4.571429 elapsed=")
    assert _mask(out.read_text()) == FORMATS_MD_RECORD
    assert best.read_text().strip() == "+-+-++--++-----+"
    rows = log.read_text().splitlines()
    assert rows[0] == "nse,elapsed_seconds,psl_best,phase_index,kind" and len(rows) == 5
    v = subprocess.run([CLI, "verify", str(best), "--histogram"], capture_output=True, text=True,
                       timeout=120)
    assert v.returncode == 0 and v.stdout.startswith("L=16 PSL=2 MF=4.571429 PSL<sqrt(L): yes")


@pytest.mark.skipif(not os.path.exists(CLI), reason="pslopt_b200 not built")
def test_cli_bench_matches_reference_readme():
    # proj/README.md:172-175: L=1023, 1e7 NSE, seeds 1-10 -> two-phase mean 28.5
    p = subprocess.run([CLI, "bench", "-L", "1023", "--runs", "10", "--max-nse", "10000000"],
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr
    assert "psl mean=28.500 min=28 max=29" in p.stdout, p.stdout


@pytest.mark.skipif(not os.path.exists(CLI), reason="pslopt_b200 not built")
def test_cli_exit_codes(tmp_path):
    r = subprocess.run([CLI, "solve", "-L", "64", "--max-nse", "100000", "--alpha2", "1100",
                        "--ls-lmt", "1"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "1100" in r.stderr and "alpha2" in r.stderr
    r = subprocess.run([CLI, "solve", "-L", "1", "--max-nse", "10"], capture_output=True, text=True)
    assert r.returncode == 1
    r = subprocess.run([CLI, "solve", "-L", "16", "--max-nse", "10", "--init",
                        str(tmp_path / "missing.txt")], capture_output=True, text=True)
    assert r.returncode == 3


@pytest.mark.skipif(not os.path.exists(CLI), reason="pslopt_b200 not built")
def test_cli_bench_over_two_contexts_matches_one():
    # the bench seeds split over two device contexts (psl_run_walks_multi, one
    # host thread each; both on GPU 0 here): the same per-seed records
    one = subprocess.run([CLI, "bench", "-L", "1023", "--runs", "10", "--max-nse", "2000000"],
                         capture_output=True, text=True, timeout=600)
    two = subprocess.run([CLI, "bench", "-L", "1023", "--runs", "10", "--max-nse", "2000000",
                          "--devices", "0,0"], capture_output=True, text=True, timeout=600)
    assert one.returncode == 0 and two.returncode == 0, one.stderr + two.stderr

    def runs(out):
        return [" ".join(w for w in ln.split() if not w.startswith("elapsed="))
                for ln in out.splitlines() if ln.startswith("run seed=")]
    assert runs(one.stdout) == runs(two.stdout) and len(runs(one.stdout)) == 10
    assert "devices=2 best seed=" in two.stdout
