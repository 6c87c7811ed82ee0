"""On-disk formats, byte-exact with the reference: HSVG velocity grids
(include/helmsweep/media.hpp:22-27, src/media.cpp:58-130) and HSFD field dumps
(src/harness.cpp:32-83). The golden files were written by the reference's own writers
(tests/golden/make_golden.py make_io). Host-only: no GPU needed."""
import os

import numpy as np
import pytest

import paper_2003_02585_b200 as hs

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def arr():
    return np.load(os.path.join(G, "io.npz"))


@pytest.mark.parametrize("name", ["io_vel2d", "io_vel3d"])
def test_velocity_grid_round_trip_is_byte_exact(arr, tmp_path, name):
    hdr, geo = arr[name + "_hdr"], arr[name + "_geo"]
    dim = int(hdr[0])
    g = hs.read_velocity_grid(os.path.join(G, name + ".hsvg"))
    assert g.dim == dim and list(g.n) == list(hdr[1:])
    np.testing.assert_array_equal(np.asarray(g.origin), geo[:3])
    np.testing.assert_array_equal(np.asarray(g.spacing), geo[3:])
    np.testing.assert_array_equal(g.c, arr[name])
    out = tmp_path / "w.hsvg"
    hs.write_velocity_grid(out, hs.VelocityGrid(dim, list(hdr[1:]), list(geo[:3]), list(geo[3:]), arr[name]))
    assert out.read_bytes() == open(os.path.join(G, name + ".hsvg"), "rb").read()


def test_field_dump_round_trip_is_byte_exact(arr, tmp_path):
    lohi, hdr = arr["io_field2d_geo"], arr["io_field2d_hdr"]
    d = hs.read_field(os.path.join(G, "io_field2d.hsfd"))
    assert d.dim == 2 and list(d.lo[:2]) == list(lohi[:2]) and list(d.hi[:2]) == list(lohi[3:5])
    np.testing.assert_array_equal(np.asarray(d.h), hdr[:3])
    np.testing.assert_array_equal(d.values, arr["io_field2d"])
    out = tmp_path / "w.hsfd"
    hs.write_field(out, 2, lohi[:3], lohi[3:], hdr[:3], hdr[3:], arr["io_field2d"])
    assert out.read_bytes() == open(os.path.join(G, "io_field2d.hsfd"), "rb").read()


def test_velocity_csv_fallback(tmp_path):
    p = tmp_path / "v.csv"
    c = np.array([1.0, 1.5, 2.0, 2.5, 3.0, 3.5], dtype=np.float32)
    p.write_text("2,3,2,0.0,0.5,0.25,0.5\n" + "\n".join(repr(float(v)) for v in c) + "\n")
    g = hs.read_velocity_csv(p)
    assert g.dim == 2 and list(g.n[:2]) == [3, 2]
    np.testing.assert_array_equal(g.c, c)
    assert g.medium(2.0).kind == "gridded"


def test_format_errors_are_data_errors(tmp_path):
    good = open(os.path.join(G, "io_vel2d.hsvg"), "rb").read()
    cases = {"magic.hsvg": b"XXXX" + good[4:], "trunc.hsvg": good[:-5],
             "version.hsvg": good[:4] + (7).to_bytes(4, "little") + good[8:]}
    for name, data in cases.items():
        (tmp_path / name).write_bytes(data)
        with pytest.raises(hs.DataError):
            hs.read_velocity_grid(tmp_path / name)
    with pytest.raises(hs.DataError):
        hs.read_velocity_grid(tmp_path / "missing.hsvg")
    with pytest.raises(hs.DataError):  # VelocityGrid::validate: non-positive sample
        hs.write_velocity_grid(tmp_path / "neg.hsvg", hs.VelocityGrid(2, [2, 2, 1], [0, 0, 0], [1, 1, 0],
                                                                      np.array([1, 1, -1, 1], np.float32)))
    fgood = open(os.path.join(G, "io_field2d.hsfd"), "rb").read()
    (tmp_path / "t.hsfd").write_bytes(fgood[:-1])
    with pytest.raises(hs.DataError):
        hs.read_field(tmp_path / "t.hsfd")
    with pytest.raises(hs.ConfigError):
        hs.write_field(tmp_path / "x.hsfd", 2, [0, 0], [2, 2], [1, 1], [0, 0], np.zeros(5, np.complex128))
