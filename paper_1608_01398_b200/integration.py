"""Switching an existing genoiht installation onto the B200.

The reference package (genoiht 0.1.0) needs no source change to run its
kernels on the device: a device ``PackedGenotypeMatrix`` satisfies the
operator protocol its ``StandardizedView.genotypes`` uses (n, p, u, v,
aty_genetic, ax_columns, decompress; reference geno_matrix.py:521-592), so
``genoiht.fit`` and friends already call the sm_100a kernels through it.
Two entry points need a dispatch to move the rest of the loop onto the
device as well:

* ``fit`` (reference iht.py:326): its O(p) host work per backtrack (top-k,
  axpy, scans; iht.py:280-285) dominates once X^T r runs on the GPU;
* ``cv_iht`` (reference model_select.py:101): its ``_fold_views``
  (model_select.py:82-98) accepts only the reference's own matrix class.

``install(genoiht)`` applies exactly the two-line dispatch INTEGRATION.md
shows for the reference source -- at run time, to an imported, unmodified
package: when ``view.genotypes`` lives on the device the call goes to this
package's ``fit`` / ``cv_iht``, otherwise to the reference's.  Every module
that bound the names at import (``genoiht``, ``genoiht.iht``,
``genoiht.model_select``, ``genoiht.simulate``, ``genoiht.cli``) is patched, so
the reference's own callers (the CLI, the experiment grid) dispatch too.
``uninstall`` restores the originals.
"""

from __future__ import annotations

import functools
import importlib

_PATCHED: dict = {}
_MODULES = ("", ".iht", ".model_select", ".simulate", ".cli")


def _on_device(view) -> bool:
    return bool(getattr(getattr(view, "genotypes", None), "is_cuda", False))


def _wrap_fit(original):
    @functools.wraps(original)
    def fit(view, y, config, warm=None):
        if _on_device(view):  # reference iht.py:326, first statement
            from .iht import fit as device_fit
            return device_fit(view, y, config, warm)
        return original(view, y, config, warm)
    fit.__wrapped_reference__ = original
    return fit


def _wrap_cv(original):
    @functools.wraps(original)
    def cv_iht(view, y, plan, config, std_mode="train", warm_start=False):
        if _on_device(view):  # reference model_select.py:101, first statement
            from .model_select import cv_iht as device_cv
            return device_cv(view, y, plan, config, std_mode, warm_start)
        return original(view, y, plan, config, std_mode, warm_start)
    cv_iht.__wrapped_reference__ = original
    return cv_iht


def install(genoiht) -> None:
    """Dispatch the imported reference package's ``fit`` and ``cv_iht`` to
    the device loop for device-resident views (idempotent)."""
    base = genoiht.__name__
    fit0 = getattr(genoiht.iht.fit, "__wrapped_reference__", genoiht.iht.fit)
    cv0 = getattr(genoiht.model_select.cv_iht, "__wrapped_reference__",
                  genoiht.model_select.cv_iht)
    fit_w, cv_w = _wrap_fit(fit0), _wrap_cv(cv0)
    for suffix in _MODULES:
        try:
            mod = importlib.import_module(base + suffix)
        except ImportError:
            continue
        for name, new in (("fit", fit_w), ("cv_iht", cv_w)):
            cur = getattr(mod, name, None)
            if cur is None:
                continue
            _PATCHED.setdefault((mod.__name__, name), getattr(cur, "__wrapped_reference__", cur))
            setattr(mod, name, new)


def uninstall(genoiht) -> None:
    """Restore the reference's own ``fit`` / ``cv_iht`` everywhere."""
    base = genoiht.__name__
    for (modname, name), original in list(_PATCHED.items()):
        if modname == base or modname.startswith(base + "."):
            setattr(importlib.import_module(modname), name, original)
            del _PATCHED[(modname, name)]
