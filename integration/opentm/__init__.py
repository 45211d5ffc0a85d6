"""``opentm`` drop-in: the reference package name backed by the B200 build.

Putting ``integration/`` on ``PYTHONPATH`` makes ``import opentm`` (and every
``opentm.<module>`` import, and ``python -m opentm``) resolve to
``paper_2405_19991_b200``, so reference-side code -- user scripts, the
``opentm_client`` bindings that shell out to ``python -m opentm``, the
reference's own test-suite -- runs on the device path unchanged
(INTEGRATION.md).  Nothing here computes; it only re-binds names.
"""

import importlib
import os
import sys

_here = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if _here not in sys.path:
    sys.path.insert(0, _here)

import paper_2405_19991_b200 as _impl  # noqa: E402
from paper_2405_19991_b200 import *  # noqa: E402,F401,F403

for _name in ("element", "field", "homogenize", "objective", "optimize", "solver", "io", "cli"):
    _mod = importlib.import_module(f"paper_2405_19991_b200.{_name}")
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod

__version__ = _impl.__version__
