"""B200-native streaming chunked block decode (Optimus, arxiv 2605.24832).

The reference package ``dllmsim`` is the caller of this path and supplies the
pieces of it that are not re-implemented here (``CommitTrace`` / ``ReplayOracle``,
the cost-model fit).  When it is not already importable, the offline install
under ``<repo>/baseline/_ref`` (``pip install --target baseline/_ref``, recipe in
``paper_2605_24832_b200/build.py``) is put on ``sys.path``.
"""

import importlib.util as _ilu
import sys as _sys
from pathlib import Path as _Path

if _ilu.find_spec("dllmsim") is None:
    _ref = _Path(__file__).resolve().parents[1] / "baseline" / "_ref"
    if (_ref / "dllmsim").is_dir():
        _sys.path.append(str(_ref))
