"""Host-side logic of the product (CPU only): lattice numbering and row
tables against the reference's meshes, and the C ABI library surface."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1902_08112_b200 import _lib, lattice
from tests.golden.specs import MESHES
from tests.helpers import oracle_levels

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


@pytest.mark.parametrize("name", list(MESHES))
def test_lattice_mesh_matches_reference_numbering(golden, name):
    g = golden["meshes"]
    blocks, n_levels, dim = MESHES[name]
    for l, lev in enumerate(lattice.build_hierarchy(blocks, n_levels, dim)):
        keys = g[f"{name}/{l}/keys"]
        assert lev.n_vertices == keys.shape[0]
        assert lev.n_cells == g[f"{name}/{l}/cells"].shape[0]
        assert np.array_equal(lev.keys, keys)
        assert np.array_equal(lev.cells, g[f"{name}/{l}/cells"])
        assert np.array_equal(lev.cell_size, g[f"{name}/{l}/cell_size"])


@pytest.mark.parametrize("name", list(MESHES))
def test_lattice_info_from_reference_style_mesh(name):
    """Row tables derived from a keys/cells mesh equal the native ones."""
    blocks, n_levels, dim = MESHES[name]
    native = lattice.build_hierarchy(blocks, n_levels, dim)
    for lev_ref, lev in zip(oracle_levels(name), native):
        a = lattice.info_from_mesh(lev_ref)
        b = lattice.info_from_mesh(lev)
        assert a.is_box == b.is_box == lev.is_box
        assert np.array_equal(a.ncell, b.ncell)
        assert a.n_vertices == b.n_vertices
        if not a.is_box:
            for x, y in zip(a.rows, b.rows):
                assert np.array_equal(x, y)
        # every cell of the mesh maps to a lattice cell; the perm is a bijection onto them
        assert np.unique(a.cell_perm).size == lev_ref.n_cells


def test_lattice_rejects_gapped_rows():
    blocks = [[(0.0, 0.0), (1.0, 1.0)], [(2.0, 0.0), (3.0, 1.0)]]
    with pytest.raises(NotImplementedError):
        lattice.LatticeMesh(blocks, 1, 2)


def _header_functions():
    src = open(os.path.join(ROOT, "include", "pffmg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pffmg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    names = _header_functions()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.exported_symbols())


def test_library_reports_argument_errors_without_a_gpu():
    lib = _lib.load()
    assert lib.pffmg_version() == 3
    rc = lib.pffmg_apply(None, None, -1, None, None, None)
    assert rc == 1
    assert b"null" in lib.pffmg_last_error()
    L = _lib.Lattice()
    L.dim = 4
    st = _lib.State()
    rc = lib.pffmg_apply(ctypes.byref(L), ctypes.byref(st), -1, None, None, None)
    assert rc == 1 and b"dim" in lib.pffmg_last_error()


def test_product_has_no_oracle_imports():
    pkg = os.path.join(ROOT, "paper_1902_08112_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f


def _integration_structs():
    """Execute the ctypes struct definitions of INTEGRATION.md's binding snippet."""
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = re.findall(r"```python\n(import ctypes as C.*?)```", doc, flags=re.S)
    assert block, "INTEGRATION.md has no ctypes binding snippet"
    src = block[0]
    defs = src[src.index("class Lattice"):src.index("lib.pffmg_apply.argtypes")]
    ns = {"C": ctypes}
    exec(defs, ns)
    return ns["Lattice"], ns["State"]


def _c_layout(tmp_path):
    """sizeof/offsetof of pffmg_lattice and pffmg_state as the C compiler lays them out."""
    fields = {"pffmg_lattice": [f for f, _ in _lib.Lattice._fields_],
              "pffmg_state": [f for f, _ in _lib.State._fields_]}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "pffmg.h"', "int main(void){"]
    for s, fs in fields.items():
        lines.append(f'printf("{s} size %zu\\n", sizeof({s}));')
        for f in fs:
            lines.append(f'printf("{s} {f} %zu\\n", offsetof({s}, {f}));')
    lines.append("return 0;}")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    lay = {}
    for line in out.splitlines():
        s, f, v = line.split()
        lay[(s, f)] = int(v)
    return lay


def test_integration_snippet_structs_match_header(tmp_path):
    """The binding INTEGRATION.md tells a maintainer to write has the header's
    layout (size and every offset), as does _lib's binding."""
    lay = _c_layout(tmp_path)
    doc_lat, doc_st = _integration_structs()
    for cname, doc_cls, lib_cls in (("pffmg_lattice", doc_lat, _lib.Lattice),
                                    ("pffmg_state", doc_st, _lib.State)):
        assert ctypes.sizeof(doc_cls) == lay[(cname, "size")] == ctypes.sizeof(lib_cls), cname
        assert [f for f, _ in doc_cls._fields_] == [f for f, _ in lib_cls._fields_], cname
        for f, _ in lib_cls._fields_:
            assert getattr(doc_cls, f).offset == lay[(cname, f)] == getattr(lib_cls, f).offset, (cname, f)


def test_struct_size_guard_rejects_foreign_layouts():
    lib = _lib.load()
    L = _lib.Lattice()
    L.dim, L.nx, L.ny, L.n_vertices = 2, 4, 4, 25
    L.struct_size = ctypes.sizeof(L) - 8          # a binding that lacks the trailing fields
    st = _lib.State()
    rc = lib.pffmg_apply(ctypes.byref(L), ctypes.byref(st), -1, None, None, None)
    assert rc == 1 and b"struct_size" in lib.pffmg_last_error()
    L.struct_size = ctypes.sizeof(L)
    st.struct_size = ctypes.sizeof(st) - 8        # the round-1 pffmg_state without phi_coef
    st.eps = 1.0
    L.hx = L.hy = 0.25
    rc = lib.pffmg_apply(ctypes.byref(L), ctypes.byref(st), -1, None, None, None)
    assert rc == 1 and b"pffmg_state.struct_size" in lib.pffmg_last_error()


@pytest.mark.parametrize("name", list(MESHES))
def test_lattice_boundary_faces_match_reference(golden, name):
    """LatticeMesh's boundary faces and tags (lattice-native) equal the
    reference's _extract_boundary + tagger arrays (mesh.py:149-161, 196-206)."""
    from tests.golden.specs import face_tagger
    g = golden["boundary"]
    blocks, n_levels, dim = MESHES[name]
    m = lattice.build_hierarchy(blocks, n_levels, dim, face_tagger)[-1]
    assert np.array_equal(m.bf_cell, g[f"{name}/bf_cell"])
    assert np.array_equal(m.bf_face, g[f"{name}/bf_face"])
    assert np.array_equal(m.bf_tag, g[f"{name}/bf_tag"])
