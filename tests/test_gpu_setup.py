"""§8(f)1: subdomain setup on the device. The extended wavenumber and the J-scaled PML CSR values
of every subdomain are computed by hs_assemble.cu; they must equal, bit for bit, the reference's own
assembly (oracle/_ref: build_coefficients + extend_to_subdomain + assemble,
/root/reference/proj/src/pml.cpp:19-52, src/media.cpp:203-217, src/operator.cpp:25-98) and the
product's host restatement (HS_HOST_SETUP=1)."""
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hs():
    import paper_2003_02585_b200 as m
    if m.device_count() == 0:
        pytest.fail("gpu test run without a CUDA device")
    return m


def _same_bits(a, b):
    return np.array_equal(a, b) and np.ascontiguousarray(a).tobytes() == np.ascontiguousarray(b).tobytes()


CASES = [
    # (name, n, parts, pad, medium keys for the reference)
    ("c1", 256, (4, 4), 20, {"media.kind": "constant", "media.kappa": 2 * math.pi * 16}),
    ("layered", 192, (3, 4), 24, {"media.kind": "two_layered", "media.kappa_down": 2 * math.pi * 12,
                                  "media.kappa_up": 2 * math.pi * 8, "media.axis": 1,
                                  "media.eta_L": 0.5 + 1 / 384, "media.epsilon": 0.0}),
    ("layered_blend", 96, (2, 3), 12, {"media.kind": "two_layered", "media.kappa_down": 30.0,
                                       "media.kappa_up": 20.0, "media.axis": 0, "media.eta_L": 0.4,
                                       "media.epsilon": 0.15}),
]


def _medium(hs, med):
    if med["media.kind"] == "constant":
        return hs.Medium("constant", kappa=med["media.kappa"])
    return hs.Medium("two_layered", kappa_down=med["media.kappa_down"], kappa_up=med["media.kappa_up"],
                     axis=med["media.axis"], eta=med["media.eta_L"], eps=med["media.epsilon"])


@pytest.mark.parametrize("name,n,parts,pad,med", CASES)
def test_device_csr_equals_reference_bitwise(hs, name, n, parts, pad, med):
    from oracle import ref
    if not ref.available():
        pytest.fail("oracle/_ref missing")
    s = hs.DdmSolver(hs.ProblemSetup(2, [n, n], list(parts), _medium(hs, med), pml_width=pad))
    r = ref.RefSolver({"dim": 2, "grid.n": [n, n], "partition": list(parts), "pml.width": pad, **med}, 4)
    exact = med["media.kind"] == "constant" or med.get("media.epsilon", 0.0) == 0.0
    for sub in range(s.nsub):
        rp, col, val = s.sub_csr(sub)
        rr, rc, rv = r.sub_csr(sub)
        assert np.array_equal(rp, rr) and np.array_equal(col, rc)
        if exact:
            assert _same_bits(val, rv), f"{name}: subdomain {sub} CSR values differ from the reference"
        else:
            # the reference build (-march=native / x86-64-v3) lets GCC contract the blend
            # kappa_down (1 - w) + kappa_up w into an FMA; the product's restatement (host and
            # device) rounds every operation: last-bit differences only
            assert np.max(np.abs(val - rv) / np.maximum(np.abs(rv), 1e-300)) <= 4e-16


def test_device_csr_equals_host_setup_gridded_3d(hs, monkeypatch, tmp_path):
    """3D and the gridded (HSVG-sampled) medium: device assembly == host assembly, bit for bit,
    and == the reference's for the gridded case."""
    from oracle import ref
    from paper_2003_02585_b200 import sources
    nl, n, pad, omega = 48, 48, 8, 2 * math.pi * 3
    c = sources.gaussian_random_velocity(nl, 11, corr_len=0.1)
    path = str(tmp_path / "v.hsvg")
    hs.write_velocity_grid(path, hs.VelocityGrid(2, [nl + 1, nl + 1, 1], [0.0, 0.0, 0.0], [1 / nl, 1 / nl, 0.0], c.ravel()))
    med = hs.Medium("gridded", velocity=c.ravel(), vel_n=(nl + 1, nl + 1, 1), vel_origin=(0.0, 0.0, 0.0),
                    vel_spacing=(1 / nl, 1 / nl, 0.0), omega=omega)
    setups = [hs.ProblemSetup(2, [n, n], [2, 3], med, pml_width=pad),
              hs.ProblemSetup(3, [12, 12, 12], [2, 1, 2], hs.Medium("constant", kappa=9.0), pml_width=4)]
    for k, st in enumerate(setups):
        dev = hs.DdmSolver(st)
        monkeypatch.setenv("HS_HOST_SETUP", "1")
        host = hs.DdmSolver(st)
        monkeypatch.delenv("HS_HOST_SETUP")
        for sub in range(dev.nsub):
            a, b = dev.sub_csr(sub), host.sub_csr(sub)
            assert all(np.array_equal(x, y) for x, y in zip(a[:2], b[:2]))
            assert _same_bits(a[2], b[2]), f"setup {k}: subdomain {sub} device and host values differ"
        if k == 0:
            r = ref.RefSolver({"dim": 2, "grid.n": [n, n], "partition": [2, 3], "pml.width": pad,
                               "media.kind": "gridded", "media.velocity_file": path, "media.omega": omega}, 4)
            for sub in range(dev.nsub):  # bilinear sampling: FMA-contracted in the reference build
                a, b = dev.sub_csr(sub)[2], r.sub_csr(sub)[2]
                assert np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)) <= 1e-14


@pytest.mark.parametrize("name", ["ddm_2d_3x2_r2", "ddm_2d_layered", "ddm_3d_2x2x2"])
def test_device_setup_plans_equal_host_setup(hs, golden, monkeypatch, name):
    """Device-built accumulate / split-source plans and CSR values give the same application, bit
    for bit, as the host-built ones (HS_HOST_SETUP=1), and the reference's u within 1e-9."""
    import ast
    z = golden(name)
    med = ast.literal_eval(str(z["medium"]))
    dim = int(z["dim"])
    st = hs.ProblemSetup(dim, [int(z["n"])] * dim, list(z["parts"]), _medium(hs, med), pml_width=int(z["pad"]))
    rounds = int(z["rounds"])
    dev = hs.DdmSolver(st)
    U = dev.ddm_solve(z["b"], rounds, None, True)
    monkeypatch.setenv("HS_HOST_SETUP", "1")
    host = hs.DdmSolver(st)
    monkeypatch.delenv("HS_HOST_SETUP")
    assert np.array_equal(U, host.ddm_solve(z["b"], rounds, None, True))
    for r in range(U.shape[0]):
        assert np.linalg.norm(U[r] - z["u"][r]) / np.linalg.norm(z["u"][r]) <= 1e-9


def test_device_global_operator_equals_host(hs, golden, monkeypatch):
    """The global operator (residual / GMRES / apply_op) assembled on the device equals the host
    assembly: A x bit for bit."""
    import ast
    z = golden("ddm_2d_layered")
    med = ast.literal_eval(str(z["medium"]))
    st = hs.ProblemSetup(2, [int(z["n"])] * 2, list(z["parts"]), _medium(hs, med), pml_width=int(z["pad"]))
    dev = hs.DdmSolver(st)
    g = np.random.default_rng(4)
    x = g.standard_normal((2, dev.global_n)) + 1j * g.standard_normal((2, dev.global_n))
    y = dev.apply_op(x)
    monkeypatch.setenv("HS_HOST_SETUP", "1")
    host = hs.DdmSolver(st)
    yh = host.apply_op(x)
    monkeypatch.delenv("HS_HOST_SETUP")
    assert np.array_equal(y, yh)
