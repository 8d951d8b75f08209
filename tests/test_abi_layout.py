"""The Python ctypes mirror (paper_2511_16665_b200/engine.py) must match the
C-ABI structs of include/tlt_b200.h byte for byte: a small C program compiled
against the header prints sizeof / offsetof of every field, compared with
the ctypes layout."""
import os
import shutil
import subprocess
import tempfile

import pytest

import paper_2511_16665_b200.engine as E

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STRUCTS = {
    "tlt_strategy": E.Strategy, "tlt_model_cfg": E.ModelCfg, "tlt_init_cfg": E.InitCfg,
    "tlt_tree_out": E.TreeOut, "tlt_tree_in": E.TreeIn, "tlt_accept_out": E.AcceptOut,
    "tlt_capture_entry": E.CaptureEntry, "tlt_cost_model": E.CostModel, "tlt_rollout_cfg": E.RolloutCfg,
    "tlt_step_metrics": E.StepMetrics, "tlt_rollout_result": E.RolloutResult,
}


@pytest.mark.skipif(shutil.which("gcc") is None, reason="no C compiler")
def test_ctypes_mirror_matches_header_layout():
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "tlt_b200.h"', 'int main(void) {']
    for cname, cls in STRUCTS.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ['return 0;', '}']
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "l.c"), os.path.join(d, "l")
        open(src, "w").write("\n".join(lines))
        subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), "-o", exe, src], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {}
    for ln in out:
        if ln:
            a, b, v = ln.split()
            got[(a, b)] = int(v)
    for cname, cls in STRUCTS.items():
        assert got[(cname, "size")] == E.C.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert got[(cname, fname)] == getattr(cls, fname).offset, (cname, fname)
