"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/er.h declares,
the Python binding mirrors the header's structs, and host-side validation (no GPU needed)
collects every error.  No compute calls are made here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "er.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:er_status|const char|int32_t|void)\s*\*?\s*(er_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def er():
    import __graft_entry__
    __graft_entry__._builder().build()
    import paper_2605_13766_b200 as er
    return er


def test_library_exports_every_declared_symbol(er):
    names = declared_functions()
    assert len(names) >= 12
    out = subprocess.run(["nm", "-D", "--defined-only", er.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (er_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert hasattr(er.lib, n)
    assert set(names) == set(er.EXPORTS)


def test_abi_version(er):
    assert er.lib.er_abi_version() == 3


def test_struct_layouts_match_header(er):
    """Compile a tiny C program against include/er.h that prints sizeof/offsetof, compare
    with the ctypes mirrors."""
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "er.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu\n", sizeof(er_batch_desc), offsetof(er_batch_desc, t0), offsetof(er_batch_desc, stream), offsetof(er_batch_desc, omega), offsetof(er_batch_desc, tile_slots));
  printf("%zu %zu %zu %zu %zu\n", sizeof(er_forcing), offsetof(er_forcing, act_component), offsetof(er_forcing, b_omega), offsetof(er_forcing, b_axis), offsetof(er_forcing, musc_component));
  printf("%zu %zu %zu\n", sizeof(er_info), offsetof(er_info, stream), offsetof(er_info, bytes_per_step));
  return 0;
}'''
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "l.c")
        open(src, "w").write(prog)
        exe = os.path.join(d, "l")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe])
        lines = subprocess.check_output([exe], text=True).split("\n")
    a = [int(x) for x in lines[0].split()]
    assert a == [C.sizeof(er.er_batch_desc), er.er_batch_desc.t0.offset, er.er_batch_desc.stream.offset,
                 er.er_batch_desc.omega.offset, er.er_batch_desc.tile_slots.offset]
    b = [int(x) for x in lines[1].split()]
    assert b == [C.sizeof(er.er_forcing), er.er_forcing.act_component.offset, er.er_forcing.b_omega.offset,
                 er.er_forcing.b_axis.offset, er.er_forcing.musc_component.offset]
    c = [int(x) for x in lines[2].split()]
    assert c == [C.sizeof(er.er_info), er.er_info.stream.offset, er.er_info.bytes_per_step.offset]


def test_host_validation_collects_all_errors(er):
    """Pure host-side validation (runs before any device work): every problem is listed."""
    d = er.er_batch_desc()
    n = np.array([3, 0, 5000], np.int32)
    mat = np.array([1.0, -2.0, 1.0])
    d.n_rods = 3
    d.n_elems = n.ctypes.data_as(C.POINTER(C.c_int32))
    d.material_per_rod = 1
    for name in ("density", "area", "I1", "I2", "youngs", "shear_mod", "alpha_c"):
        setattr(d, name, mat.ctypes.data_as(C.POINTER(C.c_double)))
    d.src_mem = 0
    with pytest.raises(er.ErError) as ei:
        er.er_create_batch(d)
    msg = str(ei.value)
    assert ei.value.status == er.ER_EINVAL
    assert "rod 1: n_elems = 0" in msg and "rod 2: n_elems = 5000" in msg


def test_null_arguments_are_rejected(er):
    assert er.lib.er_create_batch(None, None) == er.ER_EINVAL
    assert er.lib.er_step(None, 1, 1e-5) == er.ER_EINVAL
    assert er.lib.er_set_bc(None, None) == er.ER_EINVAL
    er.lib.er_destroy(None)


def test_no_oracle_in_product_path():
    """The product package never imports/links/loads the oracle (independence, task ③)."""
    pkg = os.path.join(ROOT, "paper_2605_13766_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                s = open(os.path.join(dirpath, f)).read()
                for pat in ("import oracle", "from oracle", "liboracle", "oracle.h", "orc_"):
                    assert pat not in s, (f, pat)


def test_binding_constants_mirror_header(er):
    """Every `#define ER_*` number and `ER_OPT_*` / `ER_F_*` / `ER_D_*` enumerator the binding
    exposes equals the header's value."""
    src = open(HEADER).read()
    consts = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define\s+(ER_\w+)\s+(\d+)\b", src)}
    consts.update({m.group(1): int(m.group(2)) for m in re.finditer(r"\b(ER_(?:OPT|D|F)_\w+)\s*=\s*(\d+)", src)})
    checked = 0
    for name, value in consts.items():
        if hasattr(er, name):
            assert getattr(er, name) == value, name
            checked += 1
    assert checked >= 8 and er.ER_DEFAULT_SWEEPS == consts["ER_DEFAULT_SWEEPS"]
