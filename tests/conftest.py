import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle, ORACLE_SO
    if not os.path.exists(ORACLE_SO):
        import subprocess
        subprocess.check_call(["make", "-s", "-f", os.path.join(ROOT, "oracle", "Makefile")])
    return Oracle()


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "codec_golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def reflib():
    from oracle.oracle import RefLib, REF_SO
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return RefLib()
