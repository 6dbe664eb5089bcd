"""pytest configuration: markers.  `-m "not gpu"` runs the CPU suite (oracle pins, host logic,
ABI loading, gloo multi-process); `-m gpu` runs the parity tests on a B200."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (sm_100a); parity against the float64 oracle")
    config.addinivalue_line("markers", "slow: long-running")
