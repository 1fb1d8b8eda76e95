"""B200-native Event Tensor megakernel runtime (arxiv/paper_2604_13327).

`paper_2604_13327_b200.etsim` is the drop-in for the reference's `etsim`
Python module (ref proj/python/etsim/__init__.py): graphs, lowering and the
`simulate` entry points, whose executor is the persistent sm_100a kernel.
The compiled extension is required; there is no CPU fallback.
"""

import os as _os

_HERE = _os.path.dirname(_os.path.abspath(__file__))


def _load():
    try:
        from . import _etsim  # noqa: F401  (libetgpu.so is found through the module's rpath)
    except ImportError as exc:  # pragma: no cover - a broken build must fail loudly
        raise ImportError(
            "paper_2604_13327_b200 native extension is missing; run `make` (or __graft_entry__.build())"
        ) from exc
    return _etsim


_etsim = _load()

LIBRARY_PATH = _os.path.join(_HERE, "libetgpu.so")

__all__ = ["etsim", "LIBRARY_PATH"]
