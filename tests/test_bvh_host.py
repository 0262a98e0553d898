"""Host-side pins of the wide-BVH builder (Sec. 3.1.4): conservative fp16 child
boxes ("round-to-nearest-not-lower", SPEC.md:36-44 worked values), every primitive referenced exactly
once, decoded child box contains the exact fp32 bounds of everything beneath it. No GPU needed."""
import numpy as np
import pytest

from paper_2305_20061_b200 import pt, scenes


@pytest.fixture(scope="module")
def built():
    from paper_2305_20061_b200 import _build
    _build.build()


def test_f16_not_lower_worked_values(built):
    # SPEC.md:42-44
    assert pt.f16_round(1.0, True) == 0x3C00
    assert pt.f16_round(0.0, True) == 0
    assert np.array([pt.f16_round(1.0000001, True)], np.uint16).view(np.float16)[0] == np.float16(1.0009765625)
    # brute-force f16 lattice scan on random values (incl. subnormals): smallest f16 >= x / largest <= x
    lattice = np.arange(0, 0x7C00, dtype=np.uint16).view(np.float16).astype(np.float64)
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.uniform(0, 2, 300), 10.0 ** rng.uniform(-8, 4.8, 300), lattice[rng.integers(0, 31744, 50)]])
    for x in xs:
        up = np.array([pt.f16_round(x, True)], np.uint16).view(np.float16).astype(np.float64)[0]
        dn = np.array([pt.f16_round(x, False)], np.uint16).view(np.float16).astype(np.float64)[0]
        assert up == lattice[np.searchsorted(lattice, x, side="left")]
        assert dn == lattice[np.searchsorted(lattice, x, side="right") - 1]


def _f16(bits):
    return np.array([bits & 0xFFFF], np.uint16).view(np.float16).astype(np.float32)[0]


def _check_pool(sc, pool):
    """Walk the 4-wide pool from the root; verify conservativeness and primitive coverage."""
    n_tris = sc.n_tris
    tri_lo = np.minimum(np.minimum(sc.tris["v0"], sc.tris["v1"]), sc.tris["v2"]) if n_tris else np.zeros((0, 3))
    tri_hi = np.maximum(np.maximum(sc.tris["v0"], sc.tris["v1"]), sc.tris["v2"]) if n_tris else np.zeros((0, 3))
    seen = np.zeros(n_tris + sc.n_spheres, np.int64)
    u32 = pool.view(np.uint32)
    f32 = pool.view(np.float32)

    def prim_bounds(unit):
        w = u32[unit]
        pid = int(w[3] & 0x7FFFFFFF)
        if w[3] & 0x80000000:
            c = f32[unit, :3].astype(np.float64)
            r = float(f32[unit + 1, 0])
            return pid, c - r, c + r
        return pid, tri_lo[pid].astype(np.float64), tri_hi[pid].astype(np.float64)

    def walk(unit):
        O = f32[unit, :3]
        hw = int(u32[unit, 3])
        off = hw & 0x0FFFFFFF
        # child sizes in units: nibbles in the low mantissa bits of O.x, O.y, O.z and the top of word 3
        nibs = [int(u32[unit, 0]) & 15, int(u32[unit, 1]) & 15, int(u32[unit, 2]) & 15, hw >> 28]
        words = u32[unit + 1: unit + 4].reshape(-1)
        lo_all = np.full(3, np.inf)
        hi_all = np.full(3, -np.inf)
        for ci in range(4):
            nib = nibs[ci]
            if nib == 0:
                continue
            assert nib == 4 or nib in (3, 6, 9, 12), nib
            leaf = nib != 4
            cnt = nib // 3
            w0, w1, w2 = int(words[3 * ci]), int(words[3 * ci + 1]), int(words[3 * ci + 2])
            qs = [w0, w1, w2, w0 >> 16, w1 >> 16, w2 >> 16]      # lo.x lo.y lo.z hi.x hi.y hi.z
            dlo = np.array([np.float32(O[a] + _f16(qs[a])) for a in range(3)], np.float64)
            dhi = np.array([np.float32(O[a] + _f16(qs[3 + a])) for a in range(3)], np.float64)
            if leaf:
                blo, bhi = np.full(3, np.inf), np.full(3, -np.inf)
                for k in range(cnt):
                    pid, plo, phi = prim_bounds(off + 3 * k)
                    seen[pid] += 1
                    blo, bhi = np.minimum(blo, plo), np.maximum(bhi, phi)
            else:
                blo, bhi = walk(off)
            off += nib
            assert (dlo <= blo).all() and (dhi >= bhi).all(), (dlo, blo, dhi, bhi)
            lo_all, hi_all = np.minimum(lo_all, blo), np.maximum(hi_all, bhi)
        return lo_all, hi_all

    walk(0)
    assert (seen == 1).all()


@pytest.mark.parametrize("name", ["box", "spheres", "soup", "soup_big", "tiny"])
def test_wide_bvh_conservative_and_complete(built, name):
    sc = {"box": scenes.box_scene, "spheres": scenes.spheres_scene,
          "soup": lambda: scenes.random_soup(3000, 50, 1),
          "soup_big": lambda: scenes.random_soup(2000, 0, 2, extent=300.0),
          "tiny": lambda: scenes.random_soup(1, 0, 3)}[name]()
    st, pool = pt.debug_build_bvh(sc, with_pool=True)
    assert st["leaves"] >= 1 and st["units"] % 4 == 0
    _check_pool(sc, pool)


def test_empty_scene_builds(built):
    assert pt.debug_build_bvh(scenes.empty_scene())["nodes"] == 0


def test_library_exports_every_header_symbol(built):
    import re
    import os
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "pt.h")).read()
    names = re.findall(r"PT_API\s+(?:int|const char\*)\s+(pt_\w+)\(", hdr)
    assert len(names) >= 13
    L = pt.lib()
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(pt.EXPORTED)


def test_parallel_build_is_thread_count_invariant(built):
    """The parallel builder (worker pool, chunked binning/partition of the top splits) produces the same
    pool for 1, 3 and the default number of threads (>= 2^18 primitives exercises the chunked splits)."""
    import hashlib
    import os
    sc = scenes.random_soup(300_000, 0, 7)
    digests = []
    old = os.environ.get("PT_BVH_THREADS")
    try:
        for th in ("1", "3", None):
            if th is None:
                os.environ.pop("PT_BVH_THREADS", None)
            else:
                os.environ["PT_BVH_THREADS"] = th
            st, pool = pt.debug_build_bvh(sc, with_pool=True)
            digests.append(hashlib.sha1(pool.tobytes()).hexdigest())
    finally:
        if old is None:
            os.environ.pop("PT_BVH_THREADS", None)
        else:
            os.environ["PT_BVH_THREADS"] = old
    assert len(set(digests)) == 1
    _check_pool(sc, pool) if st["units"] < 2_000_000 else None
