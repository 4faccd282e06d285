import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN_PATH = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN_PATH) as fh:
        return json.load(fh)


def oracle_args(models, gpus, policy):
    """Plain-array arguments of oracle.run for a (models, gpus, policy)."""
    stride = max(m.profile.max_batch for m in models)
    return dict(lat_ns=np.stack([m.profile.table_array(stride) for m in models]),
                max_batch=[m.profile.max_batch for m in models],
                slo_ns=[m.slo_ns for m in models],
                timeout_ns=[policy.resolve_timeout_ns(m.slo_ns) for m in models],
                n_gpus=gpus, kind=policy.kind, gather=policy.gather,
                target_batch=policy.target_batch, d_ctrl_ns=policy.d_ctrl_ns,
                d_data_ns=policy.d_data_ns)
