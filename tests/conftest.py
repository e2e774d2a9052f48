import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        return json.load(fh)


def pipeline_case(golden, idx):
    """Recorded reference pipeline run: an index into golden.json's list, or
    the name of a separately stored case (pipe_<name>.json)."""
    if isinstance(idx, int):
        return golden["pipelines"][idx]
    with open(os.path.join(GOLDEN, f"pipe_{idx}.json")) as fh:
        return json.load(fh)


PIPE_CASES = [0, 1, 2, "c1_paper"]


def golden_npz(name):
    return np.load(os.path.join(GOLDEN, name))


class ListReplay:
    """Minimal replay provider over recorded trace records (test helper)."""

    def __init__(self, records):
        self.records = records
        self.i = 0

    def propose(self, context, k, *, step=0, frontier_node=0):
        rec = self.records[self.i]
        self.i += 1
        return [(int(c["token"]), float(c["prob"])) for c in rec["candidates"]][:k]
