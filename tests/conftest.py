import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


# Measured parity values of the GPU tests (hit agreement, rel-RMSE, NIF errors) with their gates; written
# at session end to $PT_PARITY_OUT (default gpurun_out/parity.json) so the margins are on record
# (profiles/round2/parity.json is a committed copy).
_PARITY = {}


@pytest.fixture(scope="session")
def parity_log():
    def record(name, value, gate, **extra):
        d = {"value": float(value), "gate": float(gate)}
        if value:
            d["gate_over_value"] = float(gate) / float(value)
        d.update(extra)
        _PARITY[name] = d
    return record


def pytest_sessionfinish(session, exitstatus):
    if not _PARITY:
        return
    import json
    out = os.environ.get("PT_PARITY_OUT", os.path.join(ROOT, "gpurun_out", "parity.json"))
    try:
        os.makedirs(os.path.dirname(out), exist_ok=True)
        old = {}
        if os.path.exists(out):
            with open(out) as f:
                old = json.load(f)
        old.update(_PARITY)
        with open(out, "w") as f:
            json.dump(old, f, indent=1, sort_keys=True)
    except Exception:
        pass
