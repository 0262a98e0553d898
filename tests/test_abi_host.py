"""C-ABI argument validation that happens before any device work (runs without a GPU)."""
import ctypes as C

import numpy as np
import pytest

from paper_2305_20061_b200 import pt, scenes


@pytest.fixture(scope="module")
def L():
    from paper_2305_20061_b200 import _build
    _build.build()
    return pt.lib()


def _create(L, sc, n_mats=None):
    t, s, m, c = (np.ascontiguousarray(x) for x in (sc.tris, sc.spheres, sc.materials, sc.camera))
    h = C.c_void_p()
    rc = L.pt_scene_create(pt._p(t), t.shape[0], pt._p(s), s.shape[0], pt._p(m),
                           m.shape[0] if n_mats is None else n_mats, pt._p(c), C.byref(h))
    return rc, h


def test_invalid_material_index(L):
    sc = scenes.box_scene()
    rc, _ = _create(L, sc, n_mats=3)          # triangles reference materials 0..5
    assert rc == -1 and b"material" in L.pt_last_error()


def test_non_finite_vertex(L):
    sc = scenes.box_scene()
    sc.tris["v1"][3, 0] = np.nan
    rc, _ = _create(L, sc)
    assert rc == -2 and b"finite" in L.pt_last_error()


def test_bad_sphere_radius(L):
    sc = scenes.single_sphere_scene()
    sc.spheres["radius"][0] = 0.0
    rc, _ = _create(L, sc)
    assert rc == -2


def test_nif_wrong_size(L):
    b = np.zeros(100, np.uint16)
    h = C.c_void_p()
    assert L.pt_nif_load(pt._p(b), 100, C.byref(h)) == -3
    assert b"50307" in L.pt_last_error()


def test_nif_non_finite_weight(L):
    b = scenes.siren_blob(0).copy()
    b[17] = 0x7C00     # +inf
    h = C.c_void_p()
    assert L.pt_nif_load(pt._p(b), b.size, C.byref(h)) == -2


def test_null_arguments(L):
    assert L.pt_render(None, None, None, 4, 4, 1, 1, 0, None) == -1
    assert L.pt_render_async(None, None, None, 4, 4, 1, 1, 0, None, None) == -1
    assert L.pt_render_samples(None, None, None, 4, 4, 0, 1, 1, 0, 0, None, None) == -1
    assert L.pt_get_stats(None, None) == -1
    assert L.pt_version().startswith(b"pt_b200")


def test_nif_family_argument_checks(L):
    b = scenes.fourier_relu_family_blob(64, 2)
    h = C.c_void_p()
    assert L.pt_nif_load_family(96, 2, pt._p(b), b.size, C.byref(h)) == -1          # hidden % 64 != 0
    assert L.pt_nif_load_family(64, 0, pt._p(b), b.size, C.byref(h)) == -1          # layers < 1
    assert L.pt_nif_load_family(128, 2, pt._p(b), b.size, C.byref(h)) == -3         # size of (128, 2) differs
    bad = b.copy()
    bad[41] = 0x7C00
    assert L.pt_nif_load_family(64, 2, pt._p(bad), bad.size, C.byref(h)) == -2


def test_every_declared_symbol_is_exported(L):
    import re
    decl = re.findall(r"PT_API\s+[\w\s\*]+?\b(pt_\w+)\s*\(", open(pt.os.path.join(
        pt.os.path.dirname(pt._PKG), "include", "pt.h")).read())
    assert set(decl) == set(pt.EXPORTED)
    for name in decl:
        assert hasattr(L, name), name
