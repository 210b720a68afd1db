"""Drop-in aliasing: make ``import trimquad`` (and its submodules) resolve to
this package, so code written against the reference -- its own test suite
included -- runs unchanged on the B200 path.

    from paper_2101_08053_b200 import compat
    compat.install()            # before the first ``import trimquad``

Module map (reference ``pkg/src/trimquad/`` -> here): ``__init__``,
``splines``, ``quadrature``, ``trimming``, ``assembly``, ``projection``,
``cases``, ``cli``.  ``install()`` refuses to shadow a ``trimquad`` that is
already imported (mixing the two packages' objects is what the duck-typed
adapters in ``_adapt`` are for).
"""

from __future__ import annotations

import importlib
import sys

SUBMODULES = ("splines", "quadrature", "trimming", "assembly", "projection", "cases", "cli")


def install(name: str = "trimquad") -> None:
    pkg = importlib.import_module(__package__)
    cur = sys.modules.get(name)
    if cur is not None and cur is not pkg:
        raise RuntimeError(f"{name!r} is already imported from {getattr(cur, '__file__', '?')}; "
                           "install the alias before the first import")
    sys.modules[name] = pkg
    for sub in SUBMODULES:
        sys.modules[f"{name}.{sub}"] = importlib.import_module(f"{__package__}.{sub}")


def uninstall(name: str = "trimquad") -> None:
    for key in [name] + [f"{name}.{s}" for s in SUBMODULES]:
        mod = sys.modules.get(key)
        if mod is not None and getattr(mod, "__name__", "").startswith(__package__):
            del sys.modules[key]


# ---------------------------------------------------------------------------
# patch mode: keep the reference package, route its formation entry points
# (and, optionally, its constructors) to the B200 path
# ---------------------------------------------------------------------------

#: reference module -> entry points replaced by this package's
FORMATION = {"assembly": ("assemble_mass", "form_with_timings", "sum_factor_row"),
             "projection": ("assemble_rhs", "l2_error", "project", "solve_spd"),
             "quadrature": ("mass_matrix_1d",)}
#: constructors swapped too with ``constructors=True`` (the objects they
#: return are then this package's; without it the reference builds them and
#: the entry points above adapt them by duck typing, see ``_adapt``)
CONSTRUCTORS = {"trimming": ("classify_elements", "cut_cell_quadrature", "decompose_cut_element"),
                "quadrature": ("compute_wq_rules", "build_dwq", "place_wq_points")}
#: exception classes: the reference's names are rebound to these, so
#: ``except trimquad.RuleConstructionError`` catches the B200 failures and the
#: reference's own raises produce the same class
EXCEPTIONS = {"RuleConstructionError": ("quadrature", "RuleConstructionError"),
              "TrimmingConfigurationError": ("trimming", "TrimmingConfigurationError"),
              "ConditioningError": ("projection", "ConditioningError")}

_ORIGINALS = {}


def _rebind_everywhere(tq, old, new):
    """Replace every module-level binding of ``old`` in the reference package."""
    for name, mod in list(sys.modules.items()):
        if name == tq.__name__ or name.startswith(tq.__name__ + "."):
            for attr, val in list(vars(mod).items()):
                if val is old:
                    _ORIGINALS.setdefault((name, attr), old)
                    setattr(mod, attr, new)


def patch(tq, constructors: bool = False) -> None:
    """Route the reference package ``tq`` (an imported ``trimquad``) to the
    B200 path: formation entry points always, constructors on request, and
    the exception classes rebound to this package's."""
    ours = importlib.import_module(__package__)
    groups = [FORMATION] + ([CONSTRUCTORS] if constructors else [])
    for group in groups:
        for sub, names in group.items():
            ref_mod = importlib.import_module(f"{tq.__name__}.{sub}")
            our_mod = importlib.import_module(f"{__package__}.{sub}")
            for n in names:
                _rebind_everywhere(tq, getattr(ref_mod, n), getattr(our_mod, n))
    for n, (sub, attr) in EXCEPTIONS.items():
        ref_mod = importlib.import_module(f"{tq.__name__}.{sub}")
        old = getattr(ref_mod, n)
        new = getattr(importlib.import_module(f"{__package__}.{sub}"), attr)
        if old is not new:
            _rebind_everywhere(tq, old, new)
    _ = ours


def unpatch() -> None:
    """Restore every binding ``patch`` replaced."""
    for (modname, attr), old in list(_ORIGINALS.items()):
        mod = sys.modules.get(modname)
        if mod is not None:
            setattr(mod, attr, old)
    _ORIGINALS.clear()


def original(modname: str, attr: str):
    """The reference's own object behind a patched binding (for comparisons)."""
    return _ORIGINALS.get((modname, attr))
