import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA extension")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_sessionfinish(session, exitstatus):
    """GEMEL_PARITY_STATS=<path>: dump the teacher-forced admission statistics
    (tests/gpu_util.STATS) of the session as JSON (evidence for DESIGN.md R8)."""
    path = os.environ.get("GEMEL_PARITY_STATS")
    if not path:
        return
    try:
        from tests import gpu_util
    except Exception:
        return
    import json
    with open(path, "w") as f:
        json.dump(gpu_util.STATS, f)
