"""bench.py runs only on a GPU box; this CPU check catches what a first GPU run would:
names a function reads that nothing defines (e.g. a variable lost in an edit).  Every
implicitly-global name referenced in any function scope must be a module-level name, an
import, or a builtin."""
import builtins
import os
import symtable

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPTS = ["bench.py", "__graft_entry__.py", "tools/sweep.py", "tools/sweep_sgd.py",
           "tools/overlap.py", "tools/cost_model.py", "tools/ncu_summary.py",
           "tools/nvlink_counters.py", "tools/nccl_algos.py"]


def _undefined(path):
    src = open(path).read()
    top = symtable.symtable(src, path, "exec")
    module_names = {s.get_name() for s in top.get_symbols()
                    if s.is_assigned() or s.is_imported() or s.is_namespace()}
    bad = []

    def walk(t):
        for s in t.get_symbols():
            if t.get_type() != "module" and s.is_referenced() and s.is_global() \
                    and not s.is_declared_global():
                n = s.get_name()
                if n not in module_names and not hasattr(builtins, n):
                    bad.append(f"{t.get_name()}:{n}")
        for c in t.get_children():
            walk(c)

    walk(top)
    return bad


@pytest.mark.parametrize("script", SCRIPTS)
def test_no_undefined_names(script):
    path = os.path.join(ROOT, script)
    if not os.path.exists(path):
        pytest.skip(f"{script} not present")
    assert _undefined(path) == []
