"""TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference's RMHMC inner loop (arxiv 2511.06407,
package ``softabs-gp``) used as the parity checker for the CUDA path.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import it; the product package never does.

Pinned against golden vectors produced by the real reference
(``tests/golden/make_golden.py``, checked by ``tests/test_oracle_golden.py``).
"""

from .core import *  # noqa: F401,F403
