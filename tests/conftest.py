import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs on the GPU box")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_golden(name):
    path = os.path.join(ROOT, "tests", "golden", name)
    out = {}
    with open(path) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            k, v = line.split(":", 1)
            out[k.strip()] = [float(t) for t in v.split()]
    return out


@pytest.fixture
def golden():
    return load_golden


# Full-size parity metrics (tests/test_gpu_full_parity.py) are reported at the
# end of the run, so they appear in a quiet (-q) run's summary as well.
PARITY_RECORDS = []


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    if not PARITY_RECORDS:
        return
    terminalreporter.write_sep("-", "full-vector parity at BASELINE sizes (every entry vs the CPU oracle)")
    for name, worst, oracle_s in PARITY_RECORDS:
        terminalreporter.write_line(
            f"{name:10s} rel_l2 {worst['rel_l2']:.2e}  elem(RMS floor) {worst['elem_floor']:.2e}  "
            f"raw offenders {worst['raw_offenders']} (near-zero entries)  oracle {oracle_s:.1f} s")
