"""Host-side API (CPU): config parsing, residual CSV round trip, VTK writer,
mesh file I/O, synthetic mesh generators."""

import numpy as np
import pytest

from paper_2304_09485_b200.config import ConfigError, load_config, parse_patch
from paper_2304_09485_b200.driver import ResidualHistory
from paper_2304_09485_b200.mesh import MeshError, generate_box_mesh, load_mesh, save_mesh
from paper_2304_09485_b200.meshgen import generate_carved_sphere_mesh, generate_sphere_mesh, generate_wing_mesh
from paper_2304_09485_b200.output import read_residual_csv, read_vtk, write_residual_csv, write_vtk


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
    assert cfg.vtk_format == "ascii"


def test_config_output_format(tmp_path):
    ini = tmp_path / "o.ini"
    ini.write_text("[output]\ndirectory = run\nformat = Binary\n")
    assert load_config(ini).vtk_format == "binary"
    ini.write_text("[output]\nformat = hdf5\n")
    with pytest.raises(ConfigError):
        load_config(ini)


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


@pytest.mark.parametrize("split", ["tet", "hex"])
def test_vtk_binary_matches_ascii(tmp_path, split):
    mesh = generate_box_mesh((1, 1, 1), (3, 2, 2), split=split, perturb=0.1 if split == "tet" else 0.0, seed=5)
    rng = np.random.default_rng(11)
    q = np.column_stack([1 + 0.1 * rng.random(mesh.ncells), 0.1 * rng.standard_normal((mesh.ncells, 3)),
                         2.5 + 0.1 * rng.random(mesh.ncells)])
    g = rng.standard_normal((mesh.ncells, 3, 5))
    write_vtk(mesh, q, tmp_path / "a.vtk", gradients=g)
    write_vtk(mesh, q, tmp_path / "b.vtk", gradients=g, binary=True)
    a, b = read_vtk(tmp_path / "a.vtk"), read_vtk(tmp_path / "b.vtk")
    assert a.pop("encoding") == "ASCII" and b.pop("encoding") == "BINARY"
    assert a.keys() == b.keys() and "grad_rhoE" in a
    for k in a:  # %.17g round-trips float64 exactly
        assert np.array_equal(a[k], b[k]), k
    np.testing.assert_array_equal(a["points"], mesh.nodes)
    assert (tmp_path / "b.vtk").stat().st_size < (tmp_path / "a.vtk").stat().st_size


def test_vtk_mixed_cells_binary(tmp_path):
    from paper_2304_09485_b200.output import _cell_records
    sizes = np.array([4, 8, 4])
    class M:
        ncells = 3
        cell_nodes = np.arange(24).reshape(3, 8)
    rec = _cell_records(M, sizes)
    assert rec.tolist() == [4, 0, 1, 2, 3, 8, *range(8, 16), 4, 16, 17, 18, 19]


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


MESH_ARRAYS = ("nodes", "cell_nodes", "face_owner", "face_neighbor", "face_patch", "face_normal", "face_area",
               "fq_point", "cell_volume")


def _python_parse(path):
    """The reference-shaped per-line parser on its own (native reader bypassed)."""
    import paper_2304_09485_b200.mesh as M

    saved = M._load_native
    M._load_native = lambda p: None
    try:
        return M.load_mesh(path)
    finally:
        M._load_native = saved


@pytest.mark.parametrize("kind", ["tet", "hex"])
def test_native_mesh_reader_matches_python_parser(tmp_path, kind):
    m = generate_box_mesh((1, 2, 1), (3, 2, 2), split=kind, perturb=0.1 if kind == "tet" else 0.0, seed=5)
    path = tmp_path / "m.ugks"
    save_mesh(m, path)
    # comments, blank lines and stray whitespace are part of the grammar
    text = path.read_text().splitlines()
    text.insert(1, "# generated by a test")
    text.insert(3, "")
    text[5] = "  " + text[5] + "   # trailing comment"
    path.write_text("\n".join(text) + "\n")
    import paper_2304_09485_b200.mesh as M

    assert M._load_native(path) is not None  # the fast path took it
    a, b = load_mesh(path), _python_parse(path)
    for k in MESH_ARRAYS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.patch_names == b.patch_names


@pytest.mark.parametrize("bad", ["ugks-mesh 2\n", "ugks-mesh 1\nnodes 2\n0 0 0\n1 1\n",
                                 "ugks-mesh 1\nnodes 1\n0 0 x\n", "ugks-mesh 1\nnodes 0\ntets 1\n0 1 2\n"])
def test_native_mesh_reader_rejects_like_reference(tmp_path, bad):
    path = tmp_path / "bad.ugks"
    path.write_text(bad)
    import paper_2304_09485_b200.mesh as M

    assert M._load_native(path) is None
    # MeshError, or the reference's own ValueError from float() on bad numbers
    with pytest.raises(ValueError) as e1:
        load_mesh(path)
    with pytest.raises(ValueError) as e2:
        _python_parse(path)
    assert type(e1.value) is type(e2.value) and str(e1.value) == str(e2.value)
