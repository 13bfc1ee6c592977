"""CPU oracle for the FG-Attn hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU reference.  The product package (``paper_2509_16518_b200``)
never imports it and has no CPU fallback.

Pinning: every function here is checked in ``tests/test_oracle_golden.py``
against golden vectors produced by the reference package itself
(``/root/reference/pkg/src/sliceattn``, imported in the build container by
``tests/golden/make_golden.py``; the fixtures are committed under
``tests/golden/``).
"""

from .sliceattn_oracle import *  # noqa: F401,F403
