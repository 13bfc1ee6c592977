import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
GOLDEN_CASES = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libfgattn.so")
    config.addinivalue_line("markers", "slow: long-running")


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


class Golden:
    """One reference-generated fixture plus its regenerated Q/K/V."""

    def __init__(self, name):
        import oracle

        self.name = name
        z = np.load(os.path.join(GOLDEN, name + ".npz"))
        self.z = {k: z[k] for k in z.files}
        self.cfg = json.loads(str(self.z["cfg"]))
        c = self.cfg
        shape = (c["batch"], c["heads"], c["seq_len"], c["head_dim"])
        s = c["seeds"]
        self.q = oracle.gaussian(shape, s[0])
        if c["qmul"] != 1.0:
            self.q = self.q * np.float32(c["qmul"])
        self.k = oracle.gaussian(shape, s[1])
        self.v = oracle.gaussian(shape, s[2])
        for t, key in ((self.q, "q_sha"), (self.k, "k_sha"), (self.v, "v_sha")):
            assert _sha(t) == str(self.z[key]), f"{name}: regenerated {key} differs (numpy drift?)"

    @property
    def shape(self):
        c = self.cfg
        return c["batch"], c["heads"], c["seq_len"], c["head_dim"]

    @property
    def group_size(self):
        return self.cfg["group_size"]

    def lists(self, key="padded"):
        import oracle

        return oracle.padded_to_lists(self.z[key].astype(np.int32), self.group_size)

    def __getitem__(self, key):
        return self.z[key]

    def __contains__(self, key):
        return key in self.z


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = Golden(name)
        return cache[name]

    return get


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
