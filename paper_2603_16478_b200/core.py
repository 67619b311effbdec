"""Scene, state and system-matrix API of the B200 implicit step.

Mirrors the public types of the reference ``diffproj.core``
(/root/reference/pkg/src/diffproj/core.py): ``SimState`` (:23-40),
``MaterialParams`` (:43-67), ``BindingSpec`` (:70-90), ``HalfSpace``
(:93-116), ``Sphere`` (:119-143), ``Scene`` (:146-234), ``SparseMat``
(:241-288), ``SystemMatrix`` (:311-330), ``assemble_system_matrix``
(:379-389), ``predict`` (:392-397) and the JSON scene I/O (:404-485).

The host objects stay plain Python/NumPy so existing callers keep working;
``assemble_system_matrix`` uploads the scene once into a device-resident
``dp_scene`` (element kinematics, the frozen block pattern, SELL-32 system
matrix storage) owned by the returned ``SystemMatrix``.
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _lib


# ---------------------------------------------------------------------------
# state / parameters


@dataclass
class SimState:
    """Positions and velocities, flat xyz-interleaved (length 3n)."""

    q: np.ndarray
    v: np.ndarray
    step_index: int = 0

    def __post_init__(self):
        # no copy (core.py:31-33 np.asarray): a step's page-locked output
        # arrays stay page-locked as the next step's inputs
        self.q = np.asarray(self.q, dtype=np.float64).ravel()
        self.v = np.asarray(self.v, dtype=np.float64).ravel()
        if self.q.size != self.v.size:
            raise ValueError("q and v must have the same length")
        if not (np.isfinite(self.q).all() and np.isfinite(self.v).all()):
            raise ValueError("non-finite state")

    def copy(self):
        return SimState(self.q.copy(), self.v.copy(), self.step_index)

    @classmethod
    def _converged(cls, q, v, step_index):
        """The state a converged step wrote (forward_step): flat float64
        arrays whose finiteness the step already established (its residual
        at q is <= tol, a NaN or inf would have failed that test), so the
        0.5M-entry validation pass is not repeated on the host."""
        st = cls.__new__(cls)
        st.q, st.v, st.step_index = q, v, step_index
        return st


_MODELS = {"arap": 0, "neohookean": 1}


@dataclass
class MaterialParams:
    """Per-element constitutive law: ARAP (stiffness) or Neo-Hookean (E, nu)."""

    model: str = "arap"
    E: float = 1e4
    nu: float = 0.3
    stiffness: float = 1e4

    def __post_init__(self):
        if self.model not in _MODELS:
            raise ValueError(f"unknown material model {self.model!r}")
        if self.model == "neohookean":
            if not self.E > 0:
                raise ValueError("E must be positive")
            if not -1.0 < self.nu < 0.5:
                raise ValueError("nu must lie in (-1, 0.5)")
        elif self.stiffness < 0:
            raise ValueError("stiffness must be nonnegative")


@dataclass
class BindingSpec:
    """Soft attachment of one vertex to a target with compliance E_b."""

    vertex: int
    target: np.ndarray
    compliance: float = 1e-8

    def __post_init__(self):
        self.target = np.array(self.target, dtype=np.float64).reshape(-1)
        if self.target.size != 3:
            raise ValueError("binding target must be a 3-vector")
        if not self.compliance > 0:
            raise ValueError("binding compliance must be positive")

    def dofs(self):
        return 3 * int(self.vertex) + np.arange(3)


class HalfSpace:
    """Collider {x : n.x - offset >= 0} (normal normalised if needed)."""

    kind = "halfspace"

    def __init__(self, normal, offset=0.0, mu=0.0):
        n = np.array(normal, dtype=np.float64).reshape(-1)
        length = np.linalg.norm(n)
        if not np.isclose(length, 1.0, atol=1e-9):
            if length == 0:
                raise ValueError("half-space normal must be nonzero")
            n = n / length
        if mu < 0:
            raise ValueError("friction coefficient must be nonnegative")
        self.normal = n
        self.offset = float(offset)
        self.mu = float(mu)

    def gap_normal(self, x):
        return float(self.normal @ x - self.offset), self.normal

    def to_json(self):
        return {"type": "halfspace", "normal": self.normal.tolist(),
                "offset": self.offset, "mu": self.mu}


class Sphere:
    """Solid sphere collider."""

    kind = "sphere"

    def __init__(self, center, radius, mu=0.0):
        if radius <= 0:
            raise ValueError("sphere radius must be positive")
        if mu < 0:
            raise ValueError("friction coefficient must be nonnegative")
        self.center = np.array(center, dtype=np.float64).reshape(-1)
        self.radius = float(radius)
        self.mu = float(mu)

    def gap_normal(self, x):
        d = x - self.center
        r = np.linalg.norm(d)
        if r < 1e-14:
            return -self.radius, np.array([0.0, 0.0, 1.0])
        return float(r - self.radius), d / r

    def to_json(self):
        return {"type": "sphere", "center": self.center.tolist(),
                "radius": self.radius, "mu": self.mu}


@dataclass
class Scene:
    """Mesh, materials, masses, colliders, bindings and step settings.

    ``elements`` is (m,4) tetrahedra or (m,3) triangles; ``eps_fb`` stores
    2 eps^2 of the smoothed Fischer-Burmeister function.
    """

    vertices: np.ndarray
    elements: np.ndarray
    masses: np.ndarray
    materials: list = field(default_factory=list)
    gravity: np.ndarray = field(default_factory=lambda: np.array([0.0, 0.0, -9.8]))
    h: float = 0.01
    bindings: list = field(default_factory=list)
    colliders: list = field(default_factory=list)
    eps_fb: float = 1e-6
    fext: np.ndarray | None = None
    contact_activation: float = 1e-3
    # self-contact (no reference counterpart): vertices vs
    # the scene's own surface triangles frozen at the step start, friction
    # coefficient self_mu (surface_triangles, DeviceScene.sync)
    self_contact: bool = False
    self_mu: float = 0.0

    def __post_init__(self):
        self.vertices = np.array(self.vertices, dtype=np.float64).reshape(-1, 3)
        el = np.array(self.elements, dtype=np.int64)
        self.elements = el.reshape(0, 4) if el.size == 0 else el
        self.masses = np.array(self.masses, dtype=np.float64).reshape(-1)
        self.gravity = np.array(self.gravity, dtype=np.float64).reshape(-1)
        if self.fext is not None:
            self.fext = np.array(self.fext, dtype=np.float64).reshape(-1)
        self.validate()

    @property
    def n_verts(self):
        return int(self.vertices.shape[0])

    @property
    def ndof(self):
        return 3 * self.n_verts

    def mass_vector(self):
        return np.repeat(self.masses, 3)

    def external_force(self):
        g = self.mass_vector() * np.tile(self.gravity, self.n_verts)
        return g if self.fext is None else self.fext + g

    def validate(self):
        if not self.h > 0:
            raise ValueError("time step must be positive")
        if self.masses.size != self.n_verts:
            raise ValueError("masses length must match vertex count")
        if (self.masses <= 0).any():
            raise ValueError("masses must be positive")
        if not self.eps_fb > 0:
            raise ValueError("eps_fb (2*eps^2) must be positive")
        if self.elements.size and (self.elements.min() < 0
                                   or self.elements.max() >= self.n_verts):
            raise ValueError("element index out of range")
        if self.elements.shape[0] and len(self.materials) != self.elements.shape[0]:
            raise ValueError("one MaterialParams per element required")
        if self.fext is not None and self.fext.size != self.ndof:
            raise ValueError("fext length must be 3*n_verts")

    def rest_state(self):
        return SimState(self.vertices.reshape(-1).copy(), np.zeros(self.ndof))

    def copy(self):
        return Scene(
            vertices=self.vertices.copy(), elements=self.elements.copy(),
            masses=self.masses.copy(),
            materials=[MaterialParams(m.model, m.E, m.nu, m.stiffness)
                       for m in self.materials],
            gravity=self.gravity.copy(), h=self.h,
            bindings=[BindingSpec(b.vertex, b.target.copy(), b.compliance)
                      for b in self.bindings],
            colliders=[_collider_from_json(c.to_json()) for c in self.colliders],
            eps_fb=self.eps_fb,
            fext=None if self.fext is None else self.fext.copy(),
            contact_activation=self.contact_activation,
            self_contact=self.self_contact, self_mu=self.self_mu)

    # -- flattened material arrays (shared materials are cheap to expand)
    def material_arrays(self):
        mats = self.materials
        m = len(mats)
        model = np.empty(m, np.int32)
        E = np.empty(m)
        nu = np.empty(m)
        st = np.empty(m)
        cache = {}
        for i, mat in enumerate(mats):
            key = id(mat)
            row = cache.get(key)
            if row is None:
                row = (_MODELS[mat.model], mat.E, mat.nu, mat.stiffness)
                cache[key] = row
            model[i], E[i], nu[i], st[i] = row
        return model, E, nu, st


# ---------------------------------------------------------------------------
# sparse matrices (host views of device data)


class SparseMat:
    """CSR matrix with a frozen pattern (host copy; scipy-backed)."""

    def __init__(self, indptr, indices, data, shape):
        self._m = sp.csr_matrix((np.asarray(data, dtype=np.float64),
                                 np.asarray(indices, dtype=np.int64),
                                 np.asarray(indptr, dtype=np.int64)), shape=shape)
        self._m.sort_indices()

    @classmethod
    def from_scipy(cls, m):
        m = sp.csr_matrix(m)
        m.sum_duplicates()
        m.sort_indices()
        return cls(m.indptr, m.indices, m.data, m.shape)

    @classmethod
    def from_bsr(cls, rowptr, col, val, n_rows):
        """Scalar CSR from 3x3 block rows (rowptr, col, val[nnzb,3,3])."""
        b = sp.bsr_matrix((val.reshape(-1, 3, 3), col, rowptr),
                          shape=(3 * n_rows, 3 * n_rows))
        return cls.from_scipy(b.tocsr())

    indptr = property(lambda self: self._m.indptr)
    indices = property(lambda self: self._m.indices)
    data = property(lambda self: self._m.data)
    shape = property(lambda self: self._m.shape)

    def to_scipy(self):
        return self._m

    def to_dense(self):
        return self._m.toarray()

    def diagonal(self):
        return self._m.diagonal()

    def copy(self):
        return SparseMat(self.indptr.copy(), self.indices.copy(),
                         self.data.copy(), self.shape)

    def pattern_hash(self):
        return hash((self.indptr.tobytes(), self.indices.tobytes(), self.shape))


def spmv(mat, x):
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    if x.size != mat.shape[1]:
        raise ValueError("spmv dimension mismatch")
    return mat.to_scipy() @ x


def spmv_transpose(mat, x):
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    if x.size != mat.shape[0]:
        raise ValueError("spmv_transpose dimension mismatch")
    return mat.to_scipy().T @ x


# ---------------------------------------------------------------------------
# device scene


@dataclass
class Element:
    """Per-element record (reference ``elasticity.Element`` fields minus G)."""

    index: int
    verts: np.ndarray
    dofs: np.ndarray
    vol: float
    w: float
    material: object
    dim: int


def surface_triangles(elements):
    """Self-contact surface: the boundary faces of a tet mesh (faces owned by
    exactly one tet), or every triangle of a triangle mesh; (n, 3) int32."""
    el = np.asarray(elements, dtype=np.int64)
    if el.size == 0:
        return np.zeros((0, 3), np.int32)
    if el.shape[1] == 3:
        return el.astype(np.int32)
    faces = np.concatenate([el[:, [0, 1, 2]], el[:, [0, 1, 3]], el[:, [0, 2, 3]], el[:, [1, 2, 3]]])
    key = np.sort(faces, axis=1)
    _, inv, cnt = np.unique(key, axis=0, return_inverse=True, return_counts=True)
    return faces[cnt[inv.reshape(-1)] == 1].astype(np.int32)


class DeviceScene:
    """Owner of a ``dp_scene*``: element data, BSR pattern, buffers, stream."""

    def __init__(self, scene, device=0):
        L = _lib.lib()
        self.lib = L
        self.device = int(device)
        verts = _lib.f64(scene.vertices)
        els = _lib.i64(scene.elements)
        nv = els.shape[1] if els.size else 4
        model, E, nu, st = scene.material_arrays()
        masses = _lib.f64(scene.masses)
        d = _lib.SceneDesc()
        d.n_verts = scene.n_verts
        d.n_elems = els.shape[0]
        d.verts_per_elem = nv
        d.device = self.device
        d.vertices = verts.ctypes.data_as(_lib.c_double_p)
        d.elements = els.ctypes.data_as(_lib.c_int64_p)
        d.masses = masses.ctypes.data_as(_lib.c_double_p)
        d.mat_model = model.ctypes.data_as(_lib.c_int32_p)
        d.mat_E = E.ctypes.data_as(_lib.c_double_p)
        d.mat_nu = nu.ctypes.data_as(_lib.c_double_p)
        d.mat_stiffness = st.ctypes.data_as(_lib.c_double_p)
        for i in range(3):
            d.gravity[i] = float(scene.gravity[i])
        d.h = scene.h
        d.eps_fb = scene.eps_fb
        d.contact_activation = scene.contact_activation
        h = C.c_void_p()
        _lib.check(L.dp_scene_create(C.byref(d), C.byref(h)))
        self.handle = h
        self.n_verts = scene.n_verts
        self.n_elems = int(els.shape[0])
        self.verts_per_elem = nv
        self._keep = (verts, els, masses, model, E, nu, st)
        self._sync_sig = None
        self._has_fext = False
        self.sync(scene, force=True)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self.lib.dp_scene_destroy(h)
            except Exception:
                pass
            self.handle = None

    def info(self):
        inf = _lib.SceneInfo()
        _lib.check(self.lib.dp_scene_get_info(self.handle, C.byref(inf)))
        return inf

    def sync(self, scene, force=False, fext_device=None):
        """Push the per-step dynamic scene data (colliders, bindings, fext,
        h/eps/activation/gravity): the reference reads them every step."""
        L = self.lib
        cols = scene.colliders
        col_sig = tuple((c.kind, tuple(np.asarray(getattr(c, "normal", getattr(c, "center", None))).tolist()),
                         getattr(c, "offset", getattr(c, "radius", 0.0)), c.mu) for c in cols)
        bind_sig = tuple((int(b.vertex), tuple(b.target.tolist()), b.compliance) for b in scene.bindings)
        par_sig = (scene.h, scene.eps_fb, scene.contact_activation, tuple(scene.gravity.tolist()))
        fext = scene.fext
        sig = (col_sig, bind_sig, par_sig)
        prev = self._sync_sig or (None, None, None)
        if force or col_sig != prev[0]:
            n = len(cols)
            kind = np.array([0 if c.kind == "halfspace" else 1 for c in cols], np.int32)
            vec = np.array([c.normal if c.kind == "halfspace" else c.center for c in cols],
                           np.float64).reshape(-1, 3)
            sca = np.array([c.offset if c.kind == "halfspace" else c.radius for c in cols], np.float64)
            mu = np.array([c.mu for c in cols], np.float64)
            _lib.check(L.dp_scene_set_colliders(self.handle, n, _lib.ptr(kind), _lib.ptr(vec),
                                                _lib.ptr(sca), _lib.ptr(mu)))
        if force or bind_sig != prev[1]:
            nb = len(scene.bindings)
            bv = np.array([b.vertex for b in scene.bindings], np.int64)
            bt = np.array([b.target for b in scene.bindings], np.float64).reshape(-1, 3)
            bc = np.array([b.compliance for b in scene.bindings], np.float64)
            _lib.check(L.dp_scene_set_bindings(self.handle, nb, _lib.ptr(bv), _lib.ptr(bt), _lib.ptr(bc)))
        self_sig = (bool(getattr(scene, "self_contact", False)), float(getattr(scene, "self_mu", 0.0)))
        if force or self_sig != getattr(self, "_self_sig", (False, 0.0)):
            if self_sig[0]:
                if getattr(self, "_surface", None) is None:
                    self._surface = _lib.i32(surface_triangles(scene.elements).reshape(-1))
                _lib.check(L.dp_scene_set_self_contact(self.handle, self._surface.size // 3,
                                                       _lib.ptr(self._surface), self_sig[1], 1))
            elif getattr(self, "_self_sig", (False, 0.0))[0]:
                _lib.check(L.dp_scene_set_self_contact(self.handle, 0, None, 0.0, 0))
            self._self_sig = self_sig
        if force or par_sig != prev[2]:
            g = _lib.f64(scene.gravity)
            _lib.check(L.dp_scene_set_params(self.handle, scene.h, scene.eps_fb,
                                             scene.contact_activation, _lib.ptr(g)))
        # fext may be mutated in place by callers (ident setters): upload it
        # every step (or point the step at a device tensor)
        if fext_device is not None:
            _lib.check(L.dp_scene_set_fext(self.handle, _lib.ptr(fext_device), _lib.PTR_DEVICE))
        elif fext is None:
            if force or self._has_fext:
                _lib.check(L.dp_scene_set_fext(self.handle, None, _lib.PTR_HOST))
        else:
            f = _lib.f64(fext)
            _lib.check(L.dp_scene_set_fext(self.handle, _lib.ptr(f), _lib.PTR_HOST))
        self._has_fext = fext is not None or fext_device is not None
        self._sync_sig = sig

    def set_materials(self, scene):
        """Push the scene's per-element (E, nu, stiffness) to the device scene
        in place (dp_scene_set_materials): same pattern and kinematics, new
        element weights and Lame parameters."""
        _, E, nu, st = scene.material_arrays()
        _lib.check(self.lib.dp_scene_set_materials(self.handle, _lib.ptr(E), _lib.ptr(nu), _lib.ptr(st)))

    def export_bsr(self, which):
        inf = self.info()
        rowptr = np.empty(self.n_verts + 1, np.int32)
        col = np.empty(inf.nnzb, np.int32)
        val = np.empty(inf.nnzb * 9, np.float64)
        _lib.check(self.lib.dp_scene_export_bsr(self.handle, which, _lib.ptr(rowptr),
                                                _lib.ptr(col), _lib.ptr(val)))
        return SparseMat.from_bsr(rowptr, col, val, self.n_verts)

    def element_data(self):
        w = np.empty(self.n_elems)
        vol = np.empty(self.n_elems)
        _lib.check(self.lib.dp_scene_get_element_data(self.handle, _lib.ptr(w), _lib.ptr(vol)))
        return w, vol


class SystemMatrix:
    """Device-resident system matrix A = M + h^2 sum w G^T G.

    ``A`` (host SparseMat) and ``elements`` are materialised lazily; the hot
    path never leaves the device.  ``slot_map``/``diag_slots`` of the
    reference are replaced by the device contribution lists.
    """

    def __init__(self, scene, device=0):
        self.scene = scene
        self.dev = DeviceScene(scene, device)
        self._A = None
        self._elements = None

    @property
    def A(self):
        if self._A is None:
            self._A = self.dev.export_bsr(0)
        return self._A

    @property
    def elements(self):
        if self._elements is None:
            sc = self.scene
            w, vol = self.dev.element_data()
            nv = self.dev.verts_per_elem
            dim = 3 if nv == 4 else 2
            self._elements = [
                Element(index=e, verts=sc.elements[e], dofs=(3 * sc.elements[e][:, None]
                                                             + np.arange(3)).reshape(-1),
                        vol=float(vol[e]), w=float(w[e]), material=sc.materials[e], dim=dim)
                for e in range(self.dev.n_elems)]
        return self._elements

    @property
    def n_elements(self):
        return self.dev.n_elems

    def reassemble(self, scene, weights=None):
        """New weights need a new device scene (pattern is rebuilt identically)."""
        if weights is not None:
            raise NotImplementedError("per-element weight override is not supported")
        self.__init__(scene, self.dev.device)
        return self


def assemble_system_matrix(scene, device=0) -> SystemMatrix:
    """Build element kinematics, the block pattern and A on the GPU
    (reference core.assemble_system_matrix, core.py:379-389)."""
    return SystemMatrix(scene, device)


def predict(scene, state):
    """q_hat = q + h v + h^2 M^-1 (fext + m g)  (host helper, core.py:392-397)."""
    if state.q.shape[0] != scene.ndof:
        raise ValueError("state does not match scene")
    return state.q + scene.h * state.v + scene.h ** 2 * (1.0 / scene.mass_vector()) \
        * scene.external_force()


# ---------------------------------------------------------------------------
# scene JSON I/O (core.py:404-485)


def _collider_from_json(d):
    kind = d["type"].lower()
    if kind == "halfspace":
        return HalfSpace(d["normal"], d.get("offset", 0.0), d.get("mu", 0.0))
    if kind == "sphere":
        return Sphere(d["center"], d["radius"], d.get("mu", 0.0))
    raise ValueError(f"unknown collider type {d['type']!r}")


def rest_measure(vertices, el):
    """Signed tet volume (det/6) or triangle area."""
    x = vertices[np.asarray(el)]
    if len(el) == 4:
        return float(np.linalg.det(np.stack([x[1] - x[0], x[2] - x[0], x[3] - x[0]], 1))) / 6.0
    return 0.5 * float(np.linalg.norm(np.cross(x[1] - x[0], x[2] - x[0])))


def lumped_masses(vertices, elements, density):
    """Equal split of element mass (density * volume) to its vertices."""
    vertices = np.asarray(vertices, dtype=np.float64)
    elements = np.asarray(elements, dtype=np.int64)
    n = vertices.shape[0]
    if elements.size == 0:
        return np.full(n, float(density))
    x = vertices[elements]
    if elements.shape[1] == 4:
        meas = np.linalg.det(np.stack([x[:, 1] - x[:, 0], x[:, 2] - x[:, 0],
                                       x[:, 3] - x[:, 0]], axis=2)) / 6.0
    else:
        meas = 0.5 * np.linalg.norm(np.cross(x[:, 1] - x[:, 0], x[:, 2] - x[:, 0]), axis=1)
    masses = np.zeros(n)
    share = density * meas / elements.shape[1]
    for k in range(elements.shape[1]):
        np.add.at(masses, elements[:, k], share)
    masses[masses == 0] = density * 1e-6
    return masses


def scene_from_dict(doc):
    vertices = np.asarray(doc["vertices"], dtype=np.float64)
    elements = np.asarray(doc.get("elements", []), dtype=np.int64)
    if elements.size == 0:
        elements = elements.reshape(0, 4)
    if "masses" in doc:
        masses = np.asarray(doc["masses"], dtype=np.float64)
    else:
        masses = lumped_masses(vertices, elements, float(doc.get("density", 1000.0)))
    m = doc.get("material", {})
    mat = MaterialParams(model=m.get("model", "arap").lower(), E=float(m.get("E", 1e4)),
                         nu=float(m.get("nu", 0.3)), stiffness=float(m.get("stiffness", 1e4)))
    fext = doc.get("fext")
    return Scene(
        vertices=vertices, elements=elements, masses=masses,
        materials=[mat] * elements.shape[0],
        gravity=np.asarray(doc.get("gravity", [0.0, 0.0, -9.8]), dtype=np.float64),
        h=float(doc.get("dt", 0.01)),
        bindings=[BindingSpec(int(b["vertex"]), b["target"], float(b.get("compliance", 1e-8)))
                  for b in doc.get("bindings", [])],
        colliders=[_collider_from_json(c) for c in doc.get("colliders", [])],
        eps_fb=float(doc.get("eps2", 1e-6)),
        fext=None if fext is None else np.asarray(fext, dtype=np.float64).reshape(-1),
        contact_activation=float(doc.get("contact_activation", 1e-3)))


def scene_to_dict(scene):
    mat = scene.materials[0] if scene.materials else MaterialParams()
    doc = {"vertices": scene.vertices.tolist(), "elements": scene.elements.tolist(),
           "masses": scene.masses.tolist(),
           "material": {"model": mat.model, "E": mat.E, "nu": mat.nu, "stiffness": mat.stiffness},
           "gravity": scene.gravity.tolist(), "dt": scene.h, "eps2": scene.eps_fb,
           "bindings": [{"vertex": int(b.vertex), "target": b.target.tolist(),
                         "compliance": float(b.compliance)} for b in scene.bindings],
           "colliders": [c.to_json() for c in scene.colliders],
           "contact_activation": scene.contact_activation}
    if scene.fext is not None:
        doc["fext"] = scene.fext.reshape(-1, 3).tolist()
    return doc


def load_scene(path) -> Scene:
    with open(path) as f:
        return scene_from_dict(json.load(f))


def save_scene(scene, path):
    with open(path, "w") as f:
        json.dump(scene_to_dict(scene), f, indent=1)


def scene_to_arrays(scene):
    """Flat array form (the oracle / golden-fixture scene format)."""
    model, E, nu, st = scene.material_arrays()
    cols = scene.colliders
    return dict(
        vertices=scene.vertices.copy(), elements=scene.elements.copy(),
        masses=scene.masses.copy(), mat_model=model, mat_E=E, mat_nu=nu, mat_stiffness=st,
        gravity=scene.gravity.copy(), h=np.float64(scene.h), eps_fb=np.float64(scene.eps_fb),
        contact_activation=np.float64(scene.contact_activation),
        fext=np.zeros(0) if scene.fext is None else scene.fext.copy(),
        bind_vertex=np.array([b.vertex for b in scene.bindings], np.int64),
        bind_target=np.array([b.target for b in scene.bindings], np.float64).reshape(-1, 3),
        bind_compliance=np.array([b.compliance for b in scene.bindings], np.float64),
        col_kind=np.array([0 if c.kind == "halfspace" else 1 for c in cols], np.int32),
        col_vec=np.array([c.normal if c.kind == "halfspace" else c.center for c in cols],
                         np.float64).reshape(-1, 3),
        col_scalar=np.array([c.offset if c.kind == "halfspace" else c.radius for c in cols],
                            np.float64),
        col_mu=np.array([c.mu for c in cols], np.float64))


def scene_from_arrays(d):
    """Inverse of :func:`scene_to_arrays` (golden fixtures -> Scene)."""
    model = np.asarray(d["mat_model"])
    mats = [MaterialParams("neohookean" if m == 1 else "arap", float(E), float(nu), float(st))
            for m, E, nu, st in zip(model, d["mat_E"], d["mat_nu"], d["mat_stiffness"])]
    cols = []
    for k, v, s, mu in zip(d["col_kind"], d["col_vec"], d["col_scalar"], d["col_mu"]):
        cols.append(HalfSpace(v, s, mu) if k == 0 else Sphere(v, s, mu))
    fext = np.asarray(d["fext"])
    return Scene(
        vertices=d["vertices"], elements=d["elements"], masses=d["masses"], materials=mats,
        gravity=d["gravity"], h=float(d["h"]),
        bindings=[BindingSpec(int(v), t, float(c)) for v, t, c in
                  zip(d["bind_vertex"], d["bind_target"], d["bind_compliance"])],
        colliders=cols, eps_fb=float(d["eps_fb"]), fext=fext if fext.size else None,
        contact_activation=float(d["contact_activation"]))
