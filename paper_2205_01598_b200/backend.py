"""Backend seam: the CUDA backend is the only backend of this package.

The reference chooses numba or numpy at import time from LEVELMPK_BACKEND
(pkg/src/levelmpk/backend.py:21-40).  This package adds the ``cuda`` choice
the reference's seam would gain and accepts nothing
else: there is no CPU fallback, so ``numba``/``numpy`` are rejected loudly.
"""

import os

_CHOICE = os.environ.get("LEVELMPK_BACKEND", "").strip().lower()

if _CHOICE not in ("", "cuda"):
    raise RuntimeError(
        f"LEVELMPK_BACKEND={_CHOICE!r} not available in the B200 build (use 'cuda'; "
        "the CPU backends live in the reference package)"
    )

#: kept for API compatibility with levelmpk (pkg/src/levelmpk/__init__.py:12)
HAS_NUMBA = False
USING_NUMBA = False
USING_CUDA = True


def backend_name() -> str:
    return "cuda"
