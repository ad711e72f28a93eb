"""pytest plugin: run the reference's OWN tests against the B200 drop-in classes.

Loaded with ``-p dropin_plugin`` when pytest collects ``baseline/_ref/romtopt_tests`` (the
unmodified reference suite staged by tools/stage_reference.sh).  Before any test module
imports ``romtopt``, the hot-path classes are swapped exactly as INTEGRATION.md §1 shows
(HdmSolver, HelmholtzFilter, RomModel, ReducedBasis, gram_schmidt, pod in every romtopt module
that binds them), and the drop-in raises the reference's own exception classes.  Test
infrastructure only.
"""

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
for p in (REPO, REF):
    if p not in sys.path:
        sys.path.insert(0, p)


def patch():
    """Swap the hot-path classes into every romtopt module."""
    import importlib

    import romtopt

    import paper_2004_05756_b200 as tb

    mods = [importlib.import_module(f"romtopt.{m}") for m in
            ("fem", "filtering", "hdm", "rom", "problems", "trustregion", "mma", "runner")]
    hdm_cls = tb.HdmSolver
    pc, rt = os.environ.get("TB_DROPIN_PRECOND"), os.environ.get("TB_DROPIN_RTOL")
    if pc or rt:  # diagnostics: the drop-in with another preconditioner / solve tolerance
        class _Hdm(tb.HdmSolver):
            def __init__(self, *a, **kw):
                if pc:
                    kw.setdefault("preconditioner", pc)
                if rt:
                    kw.setdefault("rtol", float(rt))
                super().__init__(*a, **kw)

        hdm_cls = _Hdm
    swap = {"HdmSolver": hdm_cls, "HelmholtzFilter": tb.HelmholtzFilter, "RomModel": tb.RomModel,
            "ReducedBasis": tb.ReducedBasis, "gram_schmidt": tb.gram_schmidt, "pod": tb.pod}
    for m in mods + [romtopt]:
        for name, obj in swap.items():
            if hasattr(m, name):
                setattr(m, name, obj)
    # the drop-in raises the reference's exception types (a maintainer's integration would
    # import them from romtopt the same way)
    tb.hdm.StaleSolutionError = romtopt.hdm.StaleSolutionError
    tb.fem.IndefiniteMatrixError = romtopt.fem.IndefiniteMatrixError
    tb.rom.BasisMismatchError = romtopt.rom.BasisMismatchError
    tb.rom.DegenerateBasisError = romtopt.rom.DegenerateBasisError
    return sorted(swap)


# as a pytest plugin (-p dropin_plugin) the swap happens at import, i.e. before pytest loads the
# reference suite's conftest.py (which binds HdmSolver etc. at its own import)
if os.environ.get("TB_DROPIN_PLUGIN", "1") == "1" and "pytest" in sys.modules:
    SWAPPED = patch()
