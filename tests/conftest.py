import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Per-field gradient parity counts (fail / condition-limited / worst ratio to the 1e-3 rule)
    of the -m gpu parity tests that ran."""
    try:
        from gpu_helpers import PARITY_LOG
    except ImportError:
        return
    if PARITY_LOG:
        terminalreporter.write_sep("-", "gradient parity (SURVEY 8c.9 P4/P5): per field")
        for line in PARITY_LOG:
            terminalreporter.write_line(line)
