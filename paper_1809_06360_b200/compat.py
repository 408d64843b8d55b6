"""Binding to the reference package's own types.

The drop-in returns and raises the reference's classes whenever ``parlqr``
is importable in the caller's environment, so code written against
``parlqr`` (``except parlqr.SolverError``, ``isinstance(sol,
parlqr.LqrSolution)``) keeps working after the switch (INTEGRATION.md section
1).  This module never adds a path to ``sys.path``: ``parlqr`` is used only if
the caller's environment already provides it.  ``PLQ_NO_PARLQR=1`` forces
the stand-in classes (tests of the stand-ins).
"""

from __future__ import annotations

import importlib
import os


def reference_module(name):
    """``parlqr.<name>`` if importable (and not disabled), else None."""
    if os.environ.get("PLQ_NO_PARLQR") == "1":
        return None
    try:
        return importlib.import_module(f"parlqr.{name}")
    except ImportError:
        return None
