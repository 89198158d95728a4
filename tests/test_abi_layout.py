"""The ctypes mirror of the C-ABI structs (paper_2210_08803_b200/_lib.py) matches the
compiler's layout of include/hps_gpu.h field by field: a tiny C program built with gcc
prints sizeof/offsetof of every struct the Python host passes by pointer. CPU only."""
import json
import os
import subprocess
import tempfile

import ctypes as C
import pytest

from paper_2210_08803_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# C typedef  ->  ctypes mirror
STRUCTS = {
    "hps_table_config": L.TableConfig,
    "hps_opt_params": L.OptParams,
    "hps_cache_config": L.CacheConfig,
    "hps_cache_stats": L.CacheStats,
    "hps_update_header": L.UpdateHeader,
    "hps_slot_spec": L.SlotSpec,
    "hps_dist_config": L.DistConfig,
}


def _c_layout():
    lines = ["#include <stddef.h>", "#include <stdio.h>", '#include "hps_gpu.h"', "int main(void) {",
             '  printf("{");']
    first = True
    for cname, py in STRUCTS.items():
        fields = ", ".join(f'\\"{f}\\": %zu' for f, _ in py._fields_)
        args = ", ".join(f"offsetof({cname}, {f})" for f, _ in py._fields_)
        sep = "" if first else ", "
        first = False
        lines.append(f'  printf("{sep}\\"{cname}\\": {{\\"sizeof\\": %zu, {fields}}}", sizeof({cname}), {args});')
    lines += ['  printf("}\\n");', "  return 0;", "}"]
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "layout.c"), os.path.join(d, "layout")
        with open(src, "w") as f:
            f.write("\n".join(lines))
        subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
        return json.loads(subprocess.run([exe], check=True, capture_output=True, text=True).stdout)


@pytest.fixture(scope="module")
def layout():
    return _c_layout()


@pytest.mark.parametrize("cname", list(STRUCTS))
def test_ctypes_struct_matches_c_layout(layout, cname):
    py = STRUCTS[cname]
    c = layout[cname]
    assert C.sizeof(py) == c["sizeof"], cname
    for f, _ in py._fields_:
        assert getattr(py, f).offset == c[f], (cname, f)
