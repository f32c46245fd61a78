import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _ensure_built():
    from paper_2602_18931_b200 import build as nb
    nb.build()
    from oracle import pyoracle
    if not os.path.exists(pyoracle.LIBORACLE) or (
            os.path.isdir(pyoracle.REF_INCLUDE) and not os.path.exists(pyoracle.LIBREF)):
        pyoracle.build()


_ensure_built()


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "sim_cases.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def gpu_ctx():
    import paper_2602_18931_b200 as ws
    if ws.device_count() == 0:
        pytest.skip("no CUDA device")
    ctx = ws.Context(0)
    yield ctx
    ctx.close()
