import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_sessionfinish(session, exitstatus):
    """With PARITY_REPORT=<path>, write every compare_step's statistics (mismatched
    vs flagged near-threshold candidates, rows compared, float errors) as JSON."""
    path = os.environ.get("PARITY_REPORT")
    if not path:
        return
    try:
        import parity
    except ImportError:
        return
    if parity.REPORT:
        import json
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as f:
            json.dump(parity.REPORT, f, indent=1)
