"""Synthetic unstructured tet meshes for the sphere / wing configurations.

The reference cases (cases/sphere_*.ini, m6wing_transonic.ini) point at
external .ugks meshes that do not exist offline.  These
generators build the labelled synthetic stand-ins used by configs 2-5:

* generate_sphere_mesh -- body-fitted cubed-sphere shell between r = R and
  r = R_far (equiangular gnomonic map, geometric radial growth), each hex
  split into 24 tets through face and cell centres (conforming across the
  cube-face blocks whatever their orientation).
* generate_carved_sphere_mesh -- older stair-step stand-in: Kuhn tets on a
  stretched lattice with the sphere carved out (kept for tests).
* generate_swept_wing_mesh -- body-fitted swept, tapered wing between two
  span-end planes: O-grid around a NACA 0012 section, hexes split like the
  sphere's (config 4; the ONERA M6 geometry is not available offline).
* generate_wing_mesh -- older carved stair-step wing (kept for tests; its
  sharp corners make the transonic impulsive start fail).

Cells come out in lattice order (good locality for the device gathers).
Patch names follow the reference case files: "sphere"/"wing" for the body,
"farfield" or "inlet"/"outlet" for the box sides.
"""

from __future__ import annotations

import numpy as np

from .mesh import Mesh, MeshError

_KUHN = np.array(((0, 1, 2, 6), (0, 2, 3, 6), (0, 3, 7, 6), (0, 7, 4, 6), (0, 4, 5, 6), (0, 5, 1, 6)))
_TFACES = np.array(((0, 2, 1), (0, 1, 3), (1, 2, 3), (0, 3, 2)))


def stretched_axis(n, half, beta):
    """n cells on [-half, half] with spacing growing away from 0 (x = half sinh(b s)/sinh(b))."""
    s = np.linspace(-1.0, 1.0, n + 1)
    if beta <= 0:
        return half * s
    x = half * np.sinh(beta * s) / np.sinh(beta)
    x[0], x[-1] = -half, half
    if n % 2 == 0:
        x[n // 2] = 0.0
    return x


def _beta_for(n, half, h0):
    """Smallest stretching whose centre spacing is <= h0 (capped at 8)."""
    for b in np.linspace(0.05, 8.0, 800):
        if half * b / np.sinh(b) * 2.0 / n <= h0:
            return float(b)
    return 8.0


def _lattice(xs, ys, zs):
    nx, ny, nz = len(xs) - 1, len(ys) - 1, len(zs) - 1
    X, Y, Z = np.meshgrid(xs, ys, zs, indexing="ij")
    nodes = np.stack([X, Y, Z], axis=-1).reshape(-1, 3)

    def nid(i, j, k):
        return (i * (ny + 1) + j) * (nz + 1) + k

    i, j, k = (a.ravel() for a in np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"))
    hexes = np.stack([nid(i, j, k), nid(i + 1, j, k), nid(i + 1, j + 1, k), nid(i, j + 1, k),
                      nid(i, j, k + 1), nid(i + 1, j, k + 1), nid(i + 1, j + 1, k + 1), nid(i, j + 1, k + 1)], 1)
    return nodes, hexes[:, _KUHN].reshape(-1, 4)


def _carve(nodes, tets, inside, bounds, side_names):
    """Drop tets whose centroid is inside; classify the boundary faces of the rest."""
    cen = nodes[tets].mean(axis=1)
    keep = ~inside(cen)
    if not keep.any():
        raise MeshError("body removes every cell")
    tets = tets[keep]
    faces = tets[:, _TFACES].reshape(-1, 3)
    key = np.sort(faces, axis=1)
    kv = np.ascontiguousarray(key).view(np.dtype((np.void, 24))).ravel()
    _, inv, cnt = np.unique(kv, return_inverse=True, return_counts=True)
    bnd = faces[cnt[inv] == 1]
    p = nodes[bnd]
    lo, hi = bounds
    names = np.full(len(bnd), "", dtype=object)
    tol = 1e-9 * max(np.max(np.abs(lo)), np.max(np.abs(hi)), 1.0)
    for ax in range(3):
        names[np.all(np.abs(p[:, :, ax] - lo[ax]) < tol, axis=1)] = side_names[2 * ax]
        names[np.all(np.abs(p[:, :, ax] - hi[ax]) < tol, axis=1)] = side_names[2 * ax + 1]
    return tets, bnd, names


def _compact(nodes, tets, faces_by_patch):
    used = np.unique(tets)
    remap = -np.ones(len(nodes), dtype=np.int64)
    remap[used] = np.arange(len(used))
    return nodes[used], remap[tets], {k: remap[v] for k, v in faces_by_patch.items()}


def _tet_volumes(nodes, tets):
    p = nodes[tets]
    return np.einsum("ij,ij->i", np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), p[:, 3] - p[:, 0]) / 6.0


def _project(nodes, tets, body_nodes, target, min_frac=0.05):
    """Move body nodes to target positions unless that degrades an adjacent tet."""
    v0 = _tet_volumes(nodes, tets)
    moved = nodes.copy()
    moved[body_nodes] = target
    active = np.zeros(len(nodes), dtype=bool)
    active[body_nodes] = True
    for _ in range(20):
        v = _tet_volumes(moved, tets)
        bad = v < min_frac * v0
        if not bad.any():
            break
        revert = np.unique(tets[bad])
        revert = revert[active[revert]]
        if not len(revert):
            break
        moved[revert] = nodes[revert]
        active[revert] = False
    return moved


def _cube_dirs(n):
    """Equiangular gnomonic directions of the 6 cube faces: (6, n+1, n+1, 3) unit vectors."""
    a = np.tan(np.linspace(-np.pi / 4, np.pi / 4, n + 1))
    A, B = np.meshgrid(a, a, indexing="ij")
    one = np.ones_like(A)
    faces = [np.stack([one, A, B], -1), np.stack([-one, B, A], -1),
             np.stack([B, one, A], -1), np.stack([A, -one, B], -1),
             np.stack([A, B, one], -1), np.stack([B, A, -one], -1)]
    d = np.stack(faces)
    return d / np.linalg.norm(d, axis=-1, keepdims=True)


def _dedup_points(p, scale):
    """Unique points (rounded to 1e-12 of scale) -> (unique array, inverse index)."""
    key = np.round(p / scale * 1e12).astype(np.int64)
    kv = np.ascontiguousarray(key).view(np.dtype((np.void, 24))).ravel()
    _, first, inv = np.unique(kv, return_index=True, return_inverse=True)
    order = np.argsort(first)
    rank = np.empty_like(order)
    rank[order] = np.arange(len(order))
    return p[first[order]], rank[inv]


# quad faces of a hex (VTK order), each listed so the cell centre sees it with outward winding
_HEX_QUADS = np.array(((0, 3, 2, 1), (4, 5, 6, 7), (0, 1, 5, 4), (1, 2, 6, 5), (2, 3, 7, 6), (3, 0, 4, 7)))


def _split_hex24(corner, scale, on_wall=None, wall_centre=None):
    """Split hexes (nh, 8, 3; VTK corner order) into 24 tets each, through the
    face centres and the cell centre: conforming whatever the orientation of
    neighbouring hexes.  Face-0 centres of the hexes flagged `on_wall` are
    moved by `wall_centre` (onto the curved body).  Returns (nodes, tets,
    tri) with tri (nh, 6, 4, 3) the boundary triangles of every hex face."""
    nh = len(corner)
    # corners first; face centres then come from the deduplicated corner
    # nodes, once per unique face (both hexes of an interior face must see
    # bit-identical centres or the split is non-conforming)
    cnodes, cinv = _dedup_points(corner.reshape(-1, 3), scale)
    cid = cinv.reshape(nh, 8)
    qn_all = cid[:, _HEX_QUADS]                      # (nh, 6, 4)
    key = np.sort(qn_all.reshape(-1, 4), axis=1)
    kv = np.ascontiguousarray(key).view(np.dtype((np.void, 32))).ravel()
    _, first, finv = np.unique(kv, return_index=True, return_inverse=True)
    order = np.argsort(first)
    rank = np.empty_like(order)
    rank[order] = np.arange(len(order))
    fid_u = rank[finv].reshape(nh, 6)                # unique face id per hex face, first-occurrence order
    ukey = key[first[order]]
    fcen = cnodes[ukey].mean(axis=1)                 # (nfu, 3)
    if on_wall is not None:
        wf = np.unique(fid_u[on_wall, 0])
        fcen[wf] = wall_centre(fcen[wf])
    ccen = cnodes[cid].mean(axis=1)                  # (nh, 3)
    nodes = np.concatenate([cnodes, fcen, ccen])
    nc0, nf0 = len(cnodes), len(fcen)
    fid = nc0 + fid_u
    zid = nc0 + nf0 + np.arange(nh)
    # 24 tets: (edge a, edge b, face centre, cell centre) for each quad edge
    qn = cid[:, _HEX_QUADS]                          # (nh, 6, 4)
    a = qn
    b = np.roll(qn, -1, axis=2)
    fc = np.broadcast_to(fid[:, :, None], a.shape)
    cc = np.broadcast_to(zid[:, None, None], a.shape)
    tets = np.stack([a, b, fc, cc], axis=-1).reshape(-1, 4)
    vol = _tet_volumes(nodes, tets)
    flip = vol < 0
    tets[flip] = tets[flip][:, [0, 2, 1, 3]]
    if np.any(np.abs(vol) <= 0):
        raise MeshError("degenerate tet in a hex split")
    return nodes, tets, np.stack([a, b, fc], axis=-1)


def generate_sphere_mesh(n, radius=0.5, far=10.0, nr=None, boundary="farfield"):
    """Body-fitted synthetic tet sphere (configs 2, 3, 5): a cubed-sphere shell.

    n: cells per cube-face edge (angular), nr: radial layers (geometric growth
    from `radius` to `far`, default ~2.5 n).  Each shell hex is split into 24
    tets through its face centres and centre, which is conforming whatever the
    orientation of the neighbouring cube-face block.  About 144 n^2 nr tets.
    Patches: "sphere" (r = radius) and "farfield", or "inlet"/"outlet"
    (outer faces with x < 0 / x >= 0) for boundary="supersonic".
    """
    if nr is None:
        nr = max(4, int(round(2.5 * n)))
    dirs = _cube_dirs(n)
    g = (far / radius) ** (1.0 / nr)
    radii = radius * g ** np.arange(nr + 1)
    radii[-1] = far
    # hex corner points: (6, n+1, n+1, nr+1)
    P = dirs[:, :, :, None, :] * radii[None, None, None, :, None]
    f, i, j, k = (x.ravel() for x in np.meshgrid(np.arange(6), np.arange(n), np.arange(n), np.arange(nr),
                                                  indexing="ij"))
    corner = np.stack([P[f, i, j, k], P[f, i + 1, j, k], P[f, i + 1, j + 1, k], P[f, i, j + 1, k],
                       P[f, i, j, k + 1], P[f, i + 1, j, k + 1], P[f, i + 1, j + 1, k + 1], P[f, i, j + 1, k + 1]], 1)
    # face 0 (nodes 0-3) lies on r_k: on the wall when k == 0; its centre goes onto the sphere
    def wall_centre(fc0):
        return fc0 / np.linalg.norm(fc0, axis=1)[:, None] * radius

    nodes, tets, tri = _split_hex24(corner, far, k == 0, wall_centre)
    # boundary triangles: wall = face 0 of k == 0 hexes, far = face 1 of k == nr-1 hexes
    wall = tri[k == 0, 0].reshape(-1, 3)
    outer_tri = tri[k == nr - 1, 1].reshape(-1, 3)
    if boundary == "farfield":
        patches = {"sphere": wall, "farfield": outer_tri}
    elif boundary == "supersonic":
        xc = nodes[outer_tri].mean(axis=1)[:, 0]
        patches = {"sphere": wall, "inlet": outer_tri[xc < 0], "outlet": outer_tri[xc >= 0]}
    else:
        raise MeshError(f"unknown boundary layout {boundary!r}")
    return Mesh.build(nodes, tets, (), patches)


def _naca4_half(x, t):
    """Closed-trailing-edge NACA 4-digit half thickness at chord fraction x."""
    return 5.0 * t * (0.2969 * np.sqrt(x) - 0.1260 * x - 0.3516 * x ** 2 + 0.2843 * x ** 3 - 0.1036 * x ** 4)


def generate_swept_wing_mesh(n, span=1.5, chord=0.8, taper=0.56, sweep_deg=30.0, thickness=0.12, far=10.0,
                             nj=None, nk=None):
    """Body-fitted swept, tapered wing stand-in for config 4 (ONERA M6 geometry
    is unavailable offline): an O-grid around a NACA 00xx section (closed
    trailing edge), layered along rays from mid-chord with geometric spacing
    out to a circle of radius `far` chords, extruded over `span` with the
    section swept by `sweep_deg` and its chord tapered linearly to
    `taper` x chord at the far end; each hex split into 24 tets (conforming,
    as for the sphere).  Every grid line lies on its own ray from mid-chord,
    so the layers cannot cross.

    n: cells around the section (rounded up to a multiple of 4); nj radial
    layers (default n/2), nk spanwise layers (default n/4).  About 3 n^3 tets
    (n = 48: 331k, the size of the reference's M6 mesh).  Patches: "wing",
    "farfield", "root" and "tip" (span-end planes; slip walls in the C4 case,
    i.e. a swept wing between symmetry planes).
    """
    ni = 4 * max(2, (n + 3) // 4)
    nj = nj or max(4, ni // 2)
    nk = nk or max(2, ni // 4)
    th = np.linspace(0.0, 2.0 * np.pi, ni + 1)[:-1]
    xa = 0.5 * (1.0 + np.cos(th))                     # unit chord: TE at theta = 0, LE at pi
    ya = np.sign(np.sin(th)) * _naca4_half(xa, thickness)
    du = np.stack([xa - 0.5, ya], -1)
    ra = np.linalg.norm(du, axis=1)
    u = du / ra[:, None]                              # ray directions from mid-chord
    g = (far / 0.5) ** (1.0 / nj)
    sa = np.concatenate([[0.0], np.cumsum(g ** np.arange(nj))])
    sa /= sa[-1]                                      # 0 -> 1, geometric spacing off the wall
    r = ra[:, None] + sa[None, :] * (far - ra[:, None])   # (ni, nj+1) unit-chord radii
    zk = np.linspace(0.0, span, nk + 1)
    cz = chord * (1.0 - (1.0 - taper) * zk / span)    # local chord
    xs = zk * np.tan(np.radians(sweep_deg))           # leading-edge sweep offset
    X = (0.5 + r[:, :, None] * u[:, 0, None, None]) * cz[None, None, :] + xs[None, None, :]
    Y = (r[:, :, None] * u[:, 1, None, None]) * cz[None, None, :]
    Z = np.broadcast_to(zk[None, None, :], X.shape)
    P = np.stack([X, Y, Z], axis=-1)
    i, j, k = (x.ravel() for x in np.meshgrid(np.arange(ni), np.arange(nj), np.arange(nk), indexing="ij"))
    ip = (i + 1) % ni
    # VTK hex order: nodes 0-3 on layer j (face 0 = inner), 4-7 on j+1; face 2 at k, face 4 at k+1
    corner = np.stack([P[i, j, k], P[ip, j, k], P[ip, j, k + 1], P[i, j, k + 1],
                       P[i, j + 1, k], P[ip, j + 1, k], P[ip, j + 1, k + 1], P[i, j + 1, k + 1]], 1)
    nodes, tets, tri = _split_hex24(corner, far * chord + span)
    patches = {"wing": tri[j == 0, 0].reshape(-1, 3), "farfield": tri[j == nj - 1, 1].reshape(-1, 3),
               "root": tri[k == 0, 2].reshape(-1, 3), "tip": tri[k == nk - 1, 4].reshape(-1, 3)}
    return Mesh.build(nodes, tets, (), patches)


def generate_carved_sphere_mesh(n, radius=0.5, half=10.0, beta=None, boundary="farfield", project=True):
    """Stair-step tet sphere-in-box (legacy stand-in; see generate_sphere_mesh).

    n: lattice cells per axis (about 6 n^3 tets minus the body);
    boundary: "farfield" (all sides farfield_riemann, patch "farfield") or
    "supersonic" (x-min and lateral sides "inlet", x-max "outlet").
    """
    if beta is None:
        beta = _beta_for(n, half, radius / 10.0)  # ~10 lattice cells across the radius
    ax = stretched_axis(n, half, beta)
    nodes, tets = _lattice(ax, ax, ax)
    lo, hi = np.full(3, -half), np.full(3, half)
    sides = ("xmin", "xmax", "ymin", "ymax", "zmin", "zmax")
    tets, bnd, names = _carve(nodes, tets, lambda c: np.einsum("ij,ij->i", c, c) < radius * radius,
                              (lo, hi), sides)
    body = bnd[names == ""]
    if project:
        bn = np.unique(body)
        r = np.linalg.norm(nodes[bn], axis=1)
        nodes = _project(nodes, tets, bn, nodes[bn] * (radius / r)[:, None])
    if boundary == "farfield":
        patches = {"sphere": body, "farfield": bnd[names != ""]}
    elif boundary == "supersonic":
        patches = {"sphere": body, "inlet": bnd[(names != "") & (names != "xmax")], "outlet": bnd[names == "xmax"]}
    else:
        raise MeshError(f"unknown boundary layout {boundary!r}")
    nodes, tets, patches = _compact(nodes, tets, patches)
    return Mesh.build(nodes, tets, (), patches)


def generate_wing_mesh(n, span=1.5, root_chord=0.8, taper=0.56, sweep_deg=30.0, thickness=0.10,
                       half=8.0, beta=None):
    """Swept, tapered wing (symmetric 4-digit thickness law) stand-in for config 4.

    The wing root sits on the y = 0 plane inside the box; the body is carved
    stair-step (no projection).  Patches: "wing", "farfield".
    """
    if beta is None:
        beta = _beta_for(n, half, 0.25 * thickness * root_chord)
    ax = stretched_axis(n, half, beta)
    nodes, tets = _lattice(ax, ax, ax)
    tan_s = np.tan(np.radians(sweep_deg))

    def inside(c):
        x, y, z = c[:, 0] + 0.3, np.abs(c[:, 1]), c[:, 2]
        chord = root_chord * (1.0 - (1.0 - taper) * np.clip(y / span, 0.0, 1.0))
        xl = y * tan_s
        t = (x - xl) / chord
        ok = (y <= span) & (t >= 0.0) & (t <= 1.0)
        tc = np.clip(t, 0.0, 1.0)
        yt = 5.0 * thickness * chord * (0.2969 * np.sqrt(tc) - 0.1260 * tc - 0.3516 * tc ** 2 + 0.2843 * tc ** 3
                                         - 0.1015 * tc ** 4)
        return ok & (np.abs(z) <= yt)

    lo, hi = np.full(3, -half), np.full(3, half)
    sides = ("xmin", "xmax", "ymin", "ymax", "zmin", "zmax")
    tets, bnd, names = _carve(nodes, tets, inside, (lo, hi), sides)
    patches = {"wing": bnd[names == ""], "farfield": bnd[names != ""]}
    nodes, tets, patches = _compact(nodes, tets, patches)
    return Mesh.build(nodes, tets, (), patches)
