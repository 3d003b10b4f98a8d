"""Pins for the seeded input generator (gen/): Philox known answers, mesh closed forms, degree draw, blocks."""
import json
import math
import os

import numpy as np
import pytest

import gen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_philox_known_answers():
    # Philox4x32-10 known-answer vectors of Salmon et al. (SC'11, Random123 kat_vectors):
    # zero counter/key, all-ones counter/key, and the pi-digits counter/key.
    assert [hex(x) for x in gen.philox_raw([0, 0, 0, 0], [0, 0])] == \
        ["0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]
    assert [hex(x) for x in gen.philox_raw([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2)] == \
        ["0x408f276d", "0x41c83b0e", "0xa20bc7c6", "0x6d5451fd"]
    assert [hex(x) for x in gen.philox_raw([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344],
                                           [0xA4093822, 0x299F31D0])] == \
        ["0xd16cfe09", "0x94fdcceb", "0x5001e420", "0x24126ea1"]


@pytest.mark.parametrize("x", [1.0, 0.75, 0.5, 0.3, 1e-3, 1e-10, 2.0 ** -53, 1 - 2.0 ** -40])
def test_det_ln_matches_libm(x):
    ref = math.log(x)
    assert abs(gen.det_ln(x) - ref) <= 4e-16 * max(1.0, abs(ref))


@pytest.mark.parametrize("u", np.linspace(0, 1, 41, endpoint=False).tolist() + [0.123456789, 0.987654321])
def test_det_sincos_matches_libm(u):
    s, c = gen.det_sincos_2pi(u)
    # the libm reference rounds its argument 2*pi*u first (|arg| <= 2 pi -> ulp ~ 9e-16)
    assert abs(s - math.sin(2 * math.pi * u)) < 2e-15
    assert abs(c - math.cos(2 * math.pi * u)) < 2e-15


def test_normal_moments_and_determinism():
    z = gen.normals(0x13083995, 17, 1, 400_000)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01
    assert abs(((z ** 4).mean()) - 3.0) < 0.1
    z2 = gen.normals(0x13083995, 17, 1, 1000)
    assert np.array_equal(z[:1000], z2)
    assert not np.array_equal(z2, gen.normals(0x13083995, 18, 1, 1000))


def test_annulus_worked_example():
    g = json.load(open(os.path.join(GOLD, "annulus_1x3.json")))
    ef, fe = gen.annulus(g["nr"], g["nt"])
    assert ef.tolist() == g["elem_face"]
    assert fe.tolist() == g["face_elem"]


@pytest.mark.parametrize("nr,nt", [(1, 3), (2, 3), (2, 4), (16, 32), (64, 128)])
def test_annulus_closed_forms(nr, nt):
    ef, fe = gen.annulus(nr, nt)
    E, F = ef.shape[0], fe.shape[0]
    assert E == 2 * nr * nt
    assert F == (3 * nr + 1) * nt
    assert int((fe[:, 1] < 0).sum()) == 2 * nt         # inner + outer ring
    assert (fe[:, 0] < np.where(fe[:, 1] < 0, np.iinfo(np.int32).max, fe[:, 1])).all()   # left < right
    # each interior edge has 2 elements, each boundary edge 1; every face appears in elem_face
    cnt = np.bincount(ef.ravel(), minlength=F)
    assert (cnt == np.where(fe[:, 1] < 0, 1, 2)).all()
    for f in range(0, F, max(1, F // 50)):
        for side in (0, 1):
            e = fe[f, side]
            if e >= 0:
                assert f in ef[e]
    # faces are numbered by first encounter -> left elements are non-decreasing in face id
    assert (np.diff(fe[:, 0]) >= 0).all()


def test_degree_draw_frequencies():
    p = gen.degrees(0x13083995 + 5, 400_000, 0)
    freq = np.bincount(p, minlength=6)[1:] / len(p)
    assert np.allclose(freq, [0.1, 0.3, 0.3, 0.2, 0.1], atol=0.005)
    assert (gen.degrees(1, 10, 3) == 3).all()


@pytest.mark.parametrize("name,ne,nf", [("C1", 12, 24), ("C2", 24, 36), ("C3", 60, 60), ("C4", 120, 48)])
def test_config_sizes(name, ne, nf):
    w = gen.config(name, nr=2, nt=4)
    assert (w.elem_ne == ne).all() and (w.elem_nf == nf).all()
    assert w.uniform


def test_hp_sizes():
    w = gen.config("C5", nr=8, nt=16)
    n = (w.p + 1) * (w.p + 2) // 2
    assert (w.elem_ne == 12 * n).all()
    fe = w.face_elem
    pr = np.where(fe[:, 1] >= 0, w.p[np.maximum(fe[:, 1], 0)], w.p[fe[:, 0]])
    assert (w.face_p == np.maximum(w.p[fe[:, 0]], pr)).all()
    assert (w.face_ndof == 4 * (w.face_p + 1)).all()
    assert (w.elem_nf == w.face_ndof[w.elem_face].sum(axis=1)).all()


def test_paper_boundary_mode():
    w = gen.config("C1", nr=2, nt=4, boundary="paper")
    assert (w.face_elem[:, 1] >= 0).all()            # Gamma_h: interior edges only
    assert w.F == 3 * 2 * 4 + 4 - 2 * 4
    ring = (w.elem_face < 0).any(axis=1)
    assert ring.sum() == 2 * 4 and (w.elem_nf[ring] == 16).all() and (w.elem_nf[~ring] == 24).all()


def test_block_distributions():
    w = gen.config("C3", nr=4, nt=8)
    b = gen.host_blocks(w)
    ne, nf = 60, 60
    A = b["A"].reshape(-1, ne, ne)
    d = np.einsum("eii->ei", A)
    off = A - np.einsum("ij,ei->eij", np.eye(ne), d)
    s = 0.5 / math.sqrt(ne)
    assert abs(off.std() * math.sqrt(ne * ne / (ne * ne - ne)) - s) < 0.02 * s
    assert (d > 2 - 5 * s).all() and abs(d.mean() - (2 + math.sqrt(2 / math.pi))) < 0.05
    B = b["B"].reshape(-1, ne, nf)
    assert abs(B.std() - 1 / math.sqrt(ne)) < 0.02 / math.sqrt(ne)
    D = b["D"].reshape(-1, nf, nf)
    assert abs(np.einsum("eii->ei", D).mean() - 2.0) < 0.05
    assert abs(b["re"].std() - 1) < 0.05 and abs(b["rf"].std() - 1) < 0.05
    # a chunk regenerates exactly the same bytes
    c = gen.host_blocks(w, 5, 3)
    assert np.array_equal(c["A"], b["A"][5 * ne * ne:8 * ne * ne])
    assert np.array_equal(c["rf"], b["rf"][5 * nf:8 * nf])
