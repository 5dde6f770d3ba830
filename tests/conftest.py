import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running oracle pin (still CPU)")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.lib()
    return oracle


def pytest_sessionstart(session):
    """Build the in-tree CUDA library before any test imports the package."""
    import __graft_entry__
    __graft_entry__._builder().build()


def pytest_terminal_summary(terminalreporter):
    """Measured parity errors of every assert_parity call (floored err_q, and the raw ratio where it
    is gated), so the margins against the north_star gates are in the test log."""
    try:
        from parity import MEASURED
    except ImportError:
        return
    if not MEASURED:
        return
    tr = terminalreporter
    tr.section("parity margins (err_q floored / raw; SURVEY §8 C.6)")
    for label, tol, e, raw in MEASURED:
        parts = []
        for k in ("r", "v", "Q", "w"):
            s = f"{k} {e[k]:.1e}"
            if k in raw:
                s += f" (raw {e[k + '_raw']:.1e})"
            parts.append(s)
        worst = max([e[k] for k in ("r", "v", "Q", "w")] + [e[k + "_raw"] for k in raw])
        tr.write_line(f"{label:55s} tol {tol:.0e}  worst {worst:.1e} = {worst / tol:.2g} x tol  " + ", ".join(parts))
