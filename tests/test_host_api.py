"""Host-side API (CPU): config parsing, residual CSV round trip, VTK writer,
mesh file I/O, synthetic mesh generators."""

import numpy as np
import pytest

from paper_2304_09485_b200.config import ConfigError, load_config, parse_patch
from paper_2304_09485_b200.driver import ResidualHistory
from paper_2304_09485_b200.mesh import MeshError, generate_box_mesh, load_mesh, save_mesh
from paper_2304_09485_b200.meshgen import generate_carved_sphere_mesh, generate_sphere_mesh, generate_wing_mesh
from paper_2304_09485_b200.output import read_residual_csv, write_residual_csv, write_vtk


def test_config_defaults_and_patches(tmp_path):
    ini = tmp_path / "c.ini"
    ini.write_text("""
[mesh]
source = box
divisions = 4 4 4
split = tet
periodic = x
[scheme]
name = hweno_gmres
weights = linear
[physics]
model = viscous
mu = 0.01
reference = 1.0 0.3 0 0 0.7142857142857143
[solver]
cfl = 3.0
jacobian = frechet
[patches]
ymin = wall_noslip_isothermal lambda_wall=0.7 velocity=0.1,0,0
ymax = farfield_riemann
""")
    cfg = load_config(ini)
    assert cfg.divisions == (4, 4, 4) and cfg.periodic == ("x",)
    assert cfg.scheme == "hweno_gmres" and cfg.weights == "linear"
    assert cfg.cfl == 3.0 and cfg.krylov_dim == 10 and cfg.restarts == 3 and cfg.jacobi_sweeps == 2
    assert cfg.patches["ymin"].lambda_wall == 0.7
    assert np.allclose(cfg.patches["ymin"].velocity, [0.1, 0, 0])
    assert np.allclose(cfg.patches["ymax"].reference, cfg.reference)
    opts = cfg.solver_options()
    assert opts.jacobian == "frechet" and opts.mu == 0.01
    mesh = cfg.build_mesh()
    assert mesh.ncells == 6 * 64


def test_config_errors(tmp_path):
    with pytest.raises(ConfigError):
        load_config(tmp_path / "missing.ini")
    with pytest.raises(ConfigError):
        parse_patch("a", "wall_slip_adiabatic bogus", (1, 0, 0, 0, 1))
    with pytest.raises(ConfigError):
        parse_patch("a", "wall_noslip_isothermal", (1, 0, 0, 0, 1))


def test_residual_csv_round_trip(tmp_path):
    h = ResidualHistory()
    for k in range(5):
        h.append(k + 1, 0.1 * k, 10.0 ** -k, 2.0 * 10.0 ** -k)
    write_residual_csv(h, tmp_path / "r.csv")
    steps, t, r1, r2 = read_residual_csv(tmp_path / "r.csv")
    assert steps == h.steps and np.allclose(r1, h.res_rho_l1, rtol=1e-12) and np.allclose(r2, h.res_l2, rtol=1e-12)


def test_vtk_writer(tmp_path):
    mesh = generate_box_mesh((1, 1, 1), (2, 2, 2), split="tet")
    q = np.tile([1.0, 0.1, 0.0, 0.0, 2.5], (mesh.ncells, 1))
    write_vtk(mesh, q, tmp_path / "s.vtk", gradients=np.zeros((mesh.ncells, 3, 5)))
    text = (tmp_path / "s.vtk").read_text()
    assert f"CELLS {mesh.ncells} {5 * mesh.ncells}" in text and "VECTORS grad_rhoE double" in text
    q[0, 0] = np.nan
    with pytest.raises(ValueError):
        write_vtk(mesh, q, tmp_path / "bad.vtk")


def test_mesh_file_round_trip(tmp_path):
    m = generate_box_mesh((1, 2, 1), (2, 3, 2), split="tet", perturb=0.1, seed=3)
    save_mesh(m, tmp_path / "m.ugks")
    m2 = load_mesh(tmp_path / "m.ugks")
    assert np.array_equal(m.nodes, m2.nodes)
    assert np.array_equal(m.face_owner, m2.face_owner) and np.array_equal(m.face_neighbor, m2.face_neighbor)
    assert np.array_equal(m.face_normal, m2.face_normal)
    (tmp_path / "bad.ugks").write_text("ugks-mesh 2\n")
    with pytest.raises(MeshError):
        load_mesh(tmp_path / "bad.ugks")


def test_sphere_generator():
    m = generate_sphere_mesh(3, nr=6)
    m.validate()
    assert m.patch_names == ["sphere", "farfield"] and m.ncells == 144 * 9 * 6
    assert np.all(m.cell_volume > 0)
    wall_pts = m.fq_point[np.isin(m.fq_face, np.flatnonzero(m.face_patch == 0))]
    assert np.allclose(np.linalg.norm(wall_pts, axis=1), 0.5, rtol=0.05)
    c = generate_carved_sphere_mesh(12)
    c.validate()
    s = generate_sphere_mesh(3, boundary="supersonic")
    assert s.patch_names == ["sphere", "inlet", "outlet"]
    w = generate_wing_mesh(24)
    w.validate()
    assert int(np.sum(w.face_patch == 0)) > 0
