"""Encode the reference-generated mask of tests/golden/lens_ragged.npz (lists of length
1, 3, 127, 129, 255, 257 ...; made by tests/golden/make_golden.py from the reference
package) as an FGM1 file, the committed io fixture.  Run from the repo root."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
import oracle  # noqa: E402
from paper_2509_16518_b200 import io as fio  # noqa: E402
from paper_2509_16518_b200.sparse import SparseIndexMask  # noqa: E402

import json  # noqa: E402

z = np.load("tests/golden/lens_ragged.npz")
c = json.loads(str(z["cfg"]))
lists = oracle.padded_to_lists(z["padded"].astype(np.int32), c["group_size"])
b, h, g = c["batch"], c["heads"], -(-c["seq_len"] // c["group_size"])
nested = [[[lists[(bb * h + hh) * g + gg] for gg in range(g)] for hh in range(h)] for bb in range(b)]
mask = SparseIndexMask(b, h, c["seq_len"], c["group_size"], nested)
fio.write_mask("tests/golden/lens_ragged.fgm1", mask)
print(os.path.getsize("tests/golden/lens_ragged.fgm1"), "bytes")
