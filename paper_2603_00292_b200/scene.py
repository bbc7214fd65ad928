"""compile_scene on the GPU: flatten instances, upload, build the LBVH.

Mirrors scene.py:79-141 of the reference (``compile_scene(desc, quality)`` ->
``Scene``) with ``quality`` selecting the GPU LBVH ("lbvh30" default,
"lbvh63"; the reference's "balanced"/"fast" SAH qualities map to lbvh30).
Instances are flattened on the host into world-space fp32 triangles in
(instance, prim) order, so the reference tie rule (lowest instance, then
lowest prim; accel.py:629, 815-817) is "lowest flat id" on the device.  The
per-triangle world normal is computed reference-style in float64 (local
cross product and normalisation as in geometry.py:235-237, 274-275, then the
inverse-transpose sum and renormalisation of accel.py:843-847) and only then
rounded to fp32, which preserves the signed zeros the ONB depends on.
"""

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _native
from ._native import BuildError, check, lib, ptr
from .accel import IntersectorRegistry, SPHERE_GEOM_TYPE, sphere_data, sphere_intersector
from .camera import Camera
from .frames import frame_to_matrix, invert_affine

QUALITIES = {"lbvh30": 30, "lbvh63": 63, "balanced": 30, "fast": 30}


@dataclass
class LightTable:
    """World-space emissive triangles (sampling.py:217-253); kept for NEE ("next")."""

    v0: np.ndarray
    v1: np.ndarray
    v2: np.ndarray
    normal: np.ndarray
    emissive: np.ndarray
    area: np.ndarray
    instance: np.ndarray
    prim: np.ndarray

    def __len__(self):
        return self.v0.shape[0]


class GpuTlas:
    """Device-resident flattened scene + LBVH (replaces Tlas/TlasBundle, accel.py:439-549).

    The geometry lives on the device only (rt_scene_compile wrote it there); the host
    views ``tris``, ``tri_inst``, ``tri_prim``, ``tri_mask``, ``tri_material`` are read
    back on first use."""

    def __init__(self, ctx, handle, n, bits=30, sphere_rows=None, n_instances=None, inverses=None, build=True):
        self.ctx = ctx
        self.handle = handle
        self.n = int(n)
        self.bits = bits
        self.n_instances = n_instances
        self.inverses = inverses
        self._tris = None
        self._ids = None
        self.build_ms = None
        self.version = 0             # bumped by every (re)build: render replicas follow it
        # custom primitives: the last rows are sphere instance boxes
        self.sphere_rows = np.zeros((0, 16)) if sphere_rows is None else np.ascontiguousarray(sphere_rows, np.float64)
        self.n_spheres = int(self.sphere_rows.shape[0])
        if build:
            self.build(bits)

    def _download_ids(self):
        if self._ids is None:
            n = self.n
            ids = (np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n, np.uint32), np.empty(n, np.int32))
            check(lib().rt_scene_get_ids(self.ctx.handle, self.handle, *(ptr(x) for x in ids)))
            self._ids = ids
        return self._ids

    def geometry(self):
        """(tris (n, 9) f32, shading normals (n, 3) f32, world normals (n, 3) float64, local rows
        (n, 9) float64) of a compiled flat scene, read back from the device (parity checks)."""
        n = self.n
        out = (np.empty((n, 9), np.float32), np.empty((n, 3), np.float32), np.empty((n, 3), np.float64),
               np.empty((n, 9), np.float64))
        check(lib().rt_scene_get_geometry(self.ctx.handle, self.handle, *(ptr(x) for x in out)))
        return out

    @property
    def tri_inst(self):
        return self._download_ids()[0]

    @property
    def tri_prim(self):
        return self._download_ids()[1]

    @property
    def tri_mask(self):
        return self._download_ids()[2]

    @property
    def tri_material(self):
        return self._download_ids()[3]

    def custom_geom_types(self):
        """accel.py Tlas.custom_geom_types: geometry types of the custom BLASes present."""
        return [SPHERE_GEOM_TYPE] if self.n_spheres else []

    def build(self, bits=None, timed=False):
        """(Re)build the LBVH from the resident triangles; returns device ms if timed."""
        bits = self.bits if bits is None else bits
        ms = ctypes.c_float(-1.0)
        check(lib().rt_bvh_build(self.ctx.handle, self.handle, bits, ctypes.byref(ms) if timed else None))
        self.bits = bits
        self.version += 1
        if timed:
            self.build_ms = ms.value
            return ms.value
        return None

    @property
    def tris(self):
        """(n, 9) fp32 world triangle rows (read back from the device after a device refit)."""
        if self._tris is None:
            t = np.empty((self.n, 9), np.float32)
            check(lib().rt_scene_get_vertices(self.ctx.handle, self.handle, ptr(t)))
            self._tris = t
        return self._tris

    def refit(self, tris, bits=None):
        """New world vertices for the same triangles (Blas.refit, accel.py:263-283): H2D, the
        world normals recomputed on the device from them, rebuild."""
        tris = np.ascontiguousarray(tris, np.float32).reshape(-1, 9)
        if tris.shape[0] != self.n:
            raise ValueError(f"triangle count changed ({self.n} -> {tris.shape[0]})")
        check(lib().rt_scene_set_vertices(self.ctx.handle, self.handle, ptr(tris)))
        check(lib().rt_scene_update_normals(self.ctx.handle, self.handle))
        self._tris = tris
        self.build(bits)

    @classmethod
    def from_handle(cls, ctx, handle, n, bits, sphere_rows=None):
        """Wrap a scene built on the device (rt_tlas_flatten) whose LBVH is already built."""
        return cls(ctx, handle, n, bits, sphere_rows, build=False)

    def clone(self, device):
        """A render replica on another GPU (rt_scene_clone: device-to-device copy of the
        geometry, shading tables and built LBVH)."""
        ctx = _native.Context.get(device)
        h = ctypes.c_void_p()
        check(lib().rt_scene_clone(self.ctx.handle, self.handle, ctx.handle, ctypes.byref(h)))
        g = GpuTlas(ctx, h, self.n, self.bits, self.sphere_rows if self.n_spheres else None,
                    n_instances=self.n_instances, inverses=self.inverses, build=False)
        return g

    def build_profiled(self, bits=None):
        """Rebuild with stage events; returns dict of device ms per stage."""
        bits = self.bits if bits is None else bits
        ms = np.zeros(6, np.float32)
        check(lib().rt_bvh_build_profiled(self.ctx.handle, self.handle, bits, ptr(ms)))
        self.bits = bits
        return dict(zip(("bounds", "morton_hist", "unused", "radix_passes", "slot_init", "emit_refit"), map(float, ms)))

    def info(self):
        root = np.empty(6, np.float32)
        h = ctypes.c_int32()
        ni = ctypes.c_int64()
        check(lib().rt_bvh_info(self.ctx.handle, self.handle, ptr(root), ctypes.byref(h), ctypes.byref(ni)))
        return {"root_box": root, "height": h.value, "n_internal": ni.value}

    def download(self):
        """Full LBVH for parity checks (same layout as oracle.lbvh_build)."""
        n = self.n
        m = max(n - 1, 0)
        out = {"sorted_keys": np.empty(n, np.uint64), "order": np.empty(n, np.uint32),
               "child": np.empty((m, 2), np.int32), "parent": np.empty(max(2 * n - 1, 1), np.int32),
               "boxes": np.empty((m, 12), np.float32), "height": np.empty(m, np.int32),
               "centroid_bounds": np.empty(6, np.float32), "inv_ext": np.empty(3, np.float32)}
        check(lib().rt_bvh_download(self.ctx.handle, self.handle, ptr(out["sorted_keys"]), ptr(out["order"]),
                                    ptr(out["child"]), ptr(out["parent"]), ptr(out["boxes"]), ptr(out["height"]),
                                    ptr(out["centroid_bounds"]), ptr(out["inv_ext"]), None))
        return out

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _native._lib is not None:
                _native._lib.rt_scene_destroy(self.handle)
        except Exception:
            pass


@dataclass
class Scene:
    """scene.py:30-48; ``tlas`` is device-backed."""

    camera: Camera
    tlas: GpuTlas
    registry: IntersectorRegistry
    mat_color: np.ndarray
    mat_emissive: np.ndarray
    inst_material: np.ndarray
    lights: LightTable
    sky: np.ndarray
    background: np.ndarray
    root_box_: tuple             # (lo, hi) float64 at compile time; read through ``root_box``
    render_tlas: object = None   # two-level scenes: the device-flattened structure rt_render walks
    _meshes: dict = None         # flat scenes: mesh name -> _DeviceMesh (device refit_mesh)
    _light_src: tuple = None     # (desc, material index, instances) the light table came from
    _placements: list = None     # flat scenes: (mesh name or None, 3x4 matrix, local lo, hi) per instance
    _root_dirty: bool = False
    _render_gen: int = -1        # two-level scenes: Tlas.generation the render copy was made from
    _render_bits: int = 30
    _replicas: dict = None       # device -> (source version, render replica Scene), multi-GPU render_frame

    @property
    def root_box(self):
        """World AABB of the scene (the reference's Scene.tlas.root_box, read live: scene.py:45-48).

        Flat scenes recompute it after ``refit_mesh`` from the refitted meshes' device bounds
        (Blas.refit + refresh_instance_bounds semantics, accel.py:263-283, 477-497); two-level
        scenes read their Tlas, which ``refresh_instance_bounds`` keeps current."""
        if self.render_tlas is not None:
            return self.tlas.root_box
        if self._root_dirty:
            wlo, whi = [], []
            for name, m, lo, hi in self._placements:
                if name is not None:
                    b = self._meshes[name].device_bounds()
                    lo, hi = b[:3], b[3:]
                lo, hi = _corner_box(lo, hi, m)
                wlo.append(lo)
                whi.append(hi)
            self.root_box_ = (np.min(np.array(wlo), axis=0), np.max(np.array(whi), axis=0))
            self._root_dirty = False
        return self.root_box_

    def diagonal(self) -> float:
        lo, hi = self.root_box
        d = hi - lo
        return math.sqrt(float(d @ d))

    def replica(self, device):
        """This scene's render copy on GPU ``device`` (multi-GPU render_frame): the built flat
        structure cloned device to device, re-cloned after any rebuild or refit."""
        import dataclasses
        self.sync_render()
        src = self.render_tlas if self.render_tlas is not None else self.tlas
        if src.ctx.device == int(device):
            return self
        if self._replicas is None:
            self._replicas = {}
        hit = self._replicas.get(int(device))
        if hit is not None and hit[0] == (id(src), src.version):
            return hit[1]
        rep = dataclasses.replace(self, tlas=src.clone(int(device)), render_tlas=None, _replicas=None,
                                  root_box_=self.root_box, _root_dirty=False, _meshes=None)
        self._replicas[int(device)] = ((id(src), src.version), rep)
        return rep

    def sync_render(self):
        """Two-level scenes: bring the device-flattened render copy up to date after
        ``Tlas.refresh_instance_bounds`` (the reference re-flattens its bundle there,
        accel.py:497).  The query path reads the two-level structure directly."""
        if self.render_tlas is None or self._render_gen == self.tlas.generation:
            return
        self.tlas.flatten(self.inst_material.astype(np.int32), self.mat_color, self.mat_emissive, self.registry,
                          self._render_bits, into=self.render_tlas)
        self._render_gen = self.tlas.generation

    def refit_mesh(self, name, vertices, bits=None):
        """Blas.refit(vertices) (accel.py:263-283) for every instance of mesh `name` of a flat
        scene, on the device: the vertices go up (float64, or float32 as given: 24 or 12 B per
        vertex; the faces stay resident since compile_scene uploaded them), one kernel writes the
        instances' world triangles and world normals exactly as compile_scene does, and the
        LBVH is rebuilt.  The scene's root box and normal offset keep their compile-time values
        (the reference's flat-scene equivalent is a recompile)."""
        if self.render_tlas is not None or self._meshes is None:
            raise ValueError("refit_mesh needs a flat scene (two-level scenes refit their Blas)")
        if name not in self._meshes:
            raise ValueError(f"unknown mesh {name!r}")
        mr = self._meshes[name]
        # float32 input goes up as is (half the bytes) and is widened exactly on the device
        f32 = isinstance(vertices, np.ndarray) and vertices.dtype == np.float32
        V = np.ascontiguousarray(vertices, np.float32 if f32 else np.float64).reshape(-1, 3)
        if V.shape[0] != mr.nv:
            raise ValueError(f"vertex count changed ({mr.nv} -> {V.shape[0]})")
        tl = self.tlas
        check(lib().rt_scene_refit_mesh(tl.ctx.handle, tl.handle, mr.handle, mr.nv, ptr(V), 1 if f32 else 0))
        tl._tris = None                          # the host copy is read back on demand
        self._root_dirty = True                  # the mesh bounds were re-reduced on the device
        desc, mat_index, inst_list = self._light_src
        if any(desc.materials[d.material].has_emission for d, _ in inst_list if d.mesh == name):
            # emissive instances of this mesh: the light table follows the new vertices
            import dataclasses
            meshes = dict(desc.meshes)
            meshes[name] = dataclasses.replace(meshes[name], vertices=V.astype(np.float64))
            self._light_src = (dataclasses.replace(desc, meshes=meshes), mat_index, inst_list)
            self.lights = _light_rows(self._light_src[0], mat_index, inst_list)
            rows = np.ascontiguousarray(np.concatenate([self.lights.v0, self.lights.v1, self.lights.v2,
                                                        self.lights.normal, self.lights.emissive,
                                                        self.lights.area[:, None]], axis=1), np.float32)
            check(lib().rt_scene_set_lights(tl.ctx.handle, tl.handle, rows.shape[0], ptr(rows)))
        tl.build(bits)


class _DeviceMesh:
    """One mesh of compile_scene, resident on the device (rt_mesh_upload): the reference's
    float64 vertices and int64 faces went up once and were validated there (Blas.from_mesh's
    BuildError checks, accel.py:223-236); ``bounds`` is the float64 root box."""

    def __init__(self, ctx, V, F, wait=True):
        self.nv = int(V.shape[0])
        self.nf = int(F.shape[0])
        self.bounds = np.empty(6, np.float64)
        self._lib = lib()
        self._ctx = ctx
        h = ctypes.c_void_p()
        check(lib().rt_mesh_upload_async(ctx.handle, self.nv, ptr(V), self.nf, ptr(F), ctypes.byref(h)))
        self.handle = h
        self._src = (V, F)           # the copies read them until finish()
        if wait:
            self.finish()

    def finish(self):
        """Read the device validation back (BuildError as Blas.from_mesh) and the root box."""
        if self._src is not None:
            try:
                check(lib().rt_mesh_upload_finish(self._ctx.handle, self.handle, ptr(self.bounds)))
            finally:
                self._src = None
        return self

    def device_bounds(self):
        """float64 root box of the mesh's current vertices (re-reduced on the device by each
        refit; reading it synchronises)."""
        check(lib().rt_mesh_info(self.handle, None, None, ptr(self.bounds)))
        return self.bounds

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _native._lib is not None:
                _native._lib.rt_mesh_destroy(self.handle)
        except Exception:
            pass


class _MeshRefit:
    """One mesh of a flat scene for Scene.refit_mesh: faces + instance frames, uploaded on
    first use (rt_mesh_create)."""

    def __init__(self, nv, faces, inst, flags=0):
        self.nv = int(nv)
        self.flags = int(flags)
        self.faces = np.ascontiguousarray(faces, np.int32).reshape(-1, 3)
        # rows of 21 doubles: the 3x4 matrix, then the 3x3 block of its inverse
        self.xform = np.ascontiguousarray([np.concatenate([m.reshape(12), inv[:, :3].reshape(9)]) for m, inv, _ in inst],
                                          np.float64)
        self.offset = np.ascontiguousarray([o for _, _, o in inst], np.int64)
        self._h = None

    def handle(self, ctx):
        if self._h is None:
            h = ctypes.c_void_p()
            check(lib().rt_mesh_create(ctx.handle, self.nv, self.faces.shape[0], ptr(self.faces), len(self.offset),
                                       ptr(self.xform), ptr(self.offset), self.flags, ctypes.byref(h)))
            self._h = h
        return self._h

    def __del__(self):
        try:
            if self._h and _native._lib is not None:
                _native._lib.rt_mesh_destroy(self._h)
        except Exception:
            pass


def _light_rows(desc, mats_index, inst_list):
    """scene.py:58-76."""
    rows = []
    for i, (decl, m) in enumerate(inst_list):
        mat = desc.materials[decl.material]
        if not mat.has_emission:
            continue
        mesh = desc.meshes[decl.mesh]
        world = mesh.vertices @ m[:, :3].T + m[:, 3]
        for prim, (i0, i1, i2) in enumerate(mesh.faces):
            w0, w1, w2 = world[i0], world[i1], world[i2]
            n = np.cross(w1 - w0, w2 - w1)
            nlen = math.sqrt(float(n @ n))
            if nlen == 0.0:
                continue
            rows.append((w0, w1, w2, n / nlen, mat.emissive, 0.5 * nlen, i, prim))
    if not rows:
        z = np.zeros((0, 3))
        return LightTable(z, z, z, z, z, np.zeros(0), np.zeros(0, np.int64), np.zeros(0, np.int64))
    col = lambda k: np.array([r[k] for r in rows])
    return LightTable(col(0).reshape(-1, 3), col(1).reshape(-1, 3), col(2).reshape(-1, 3), col(3).reshape(-1, 3),
                      col(4).reshape(-1, 3), col(5), col(6).astype(np.int64), col(7).astype(np.int64))


def compile_scene(desc, quality: str = "lbvh30", device: int = 0, two_level: bool = False) -> Scene:
    """Flatten + upload + LBVH build (scene.py:79-141 semantics, GPU backend).

    two_level=True builds the reference's structure instead -- one device Blas per mesh
    (and per sphere), a Tlas over the instances -- so queries run the two-level kernels;
    rendering walks a flattened copy made on the device from that Tlas."""
    if quality not in QUALITIES:
        raise ValueError(f"unknown build quality {quality!r}, expected one of {tuple(QUALITIES)}")
    if two_level:
        return _compile_two_level(desc, quality, device)
    mat_names = list(desc.materials)
    mat_index = {n: i for i, n in enumerate(mat_names)}
    mat_color = np.array([desc.materials[n].color for n in mat_names]).reshape(-1, 3)
    mat_emissive = np.array([desc.materials[n].emissive for n in mat_names]).reshape(-1, 3)
    if not desc.instances and not desc.spheres:
        raise BuildError("a scene needs at least one instance")
    ctx = _native.Context.get(device)

    # every mesh up once, validated on the device (Blas.from_mesh, accel.py:223-236)
    mesh_names = list(desc.meshes)
    dmeshes = {}
    for name in mesh_names:
        mesh = desc.meshes[name]
        V = np.ascontiguousarray(mesh.vertices, np.float64).reshape(-1, 3)
        F = np.ascontiguousarray(mesh.faces, np.int64).reshape(-1, 3)
        try:
            dmeshes[name] = _DeviceMesh(ctx, V, F, wait=False)   # validated below, after the host-side tables
        except Exception:
            for dm in dmeshes.values():                          # earlier meshes' verdicts come first
                dm.finish()
            raise

    # host-side tables while the meshes cross PCIe; any error here is raised after the
    # meshes' own verdicts, as the reference builds every Blas before the instances
    try:
        # sphere instances after the mesh instances (scene.py:101-112): one custom primitive
        # each, flat ids after every triangle; its leaf box is the world AABB of the
        # transformed local box (accel.py:459-469), rounded outward to fp32
        n_sph = len(desc.spheres) if desc.spheres else 0
        customs = (_native.CustomSrc * max(n_sph, 1))()
        sph_rows, sph_boxes = [], []
        if n_sph:
            rows = np.array([[*sph.center, sph.radius] for sph in desc.spheres], dtype=np.float64)
            sphere_data(rows)                               # radius > 0 (accel.py:403-408)
            for k, sph in enumerate(desc.spheres):
                m = frame_to_matrix(sph.frame)
                try:
                    inv = invert_affine(m)
                except ValueError as exc:
                    raise BuildError(f"sphere {k} frame is not invertible") from exc
                c, r = rows[k, :3], rows[k, 3]
                lo, hi = _corner_box(c - r, c + r, m)
                lo32, hi32 = lo.astype(np.float32), hi.astype(np.float32)
                lo32 = np.where(lo32.astype(np.float64) > lo, np.nextafter(lo32, np.float32(-np.inf)), lo32)
                hi32 = np.where(hi32.astype(np.float64) < hi, np.nextafter(hi32, np.float32(np.inf)), hi32)
                row = np.concatenate([inv.reshape(12), c, [r]])
                cs = customs[k]
                cs.box[:] = [float(x) for x in np.concatenate([lo32, hi32, lo32])]
                cs.material = mat_index[sph.material]
                cs.mask = int(sph.mask)
                cs.row[:] = [float(x) for x in row]
                sph_rows.append(row)
                sph_boxes.append((lo, hi, inv, c - r, c + r, m))

        # instances (Instance + Tlas frames, accel.py:339-346, 451-472)
        n_inst = len(desc.instances)
        srcs = (_native.InstanceSrc * max(n_inst, 1))()
        inst_material, inst_list, inverses, placements = [], [], [], []
        wlo, whi = [], []
        for i, decl in enumerate(desc.instances):
            m = frame_to_matrix(decl.frame)
            try:
                inv = invert_affine(m)
            except ValueError as exc:
                raise BuildError(f"instance {i} frame is not invertible") from exc
            inverses.append(inv)
            inst_list.append((decl, m))
            placements.append((decl.mesh, m, None, None))
            mi = mat_index[decl.material]
            inst_material.append(mi)
            src = srcs[i]
            src.mesh = mesh_names.index(decl.mesh)
            src.material = mi
            src.mask = int(decl.mask)
            src.matrix[:] = [float(x) for x in m.reshape(12)]
            src.inverse[:] = [float(x) for x in inv.reshape(12)]
    except Exception:
        for name in mesh_names:
            dmeshes[name].finish()
        raise

    # the flat scene written on the device behind the meshes' validation (nothing is written
    # for a mesh that fails it), then the verdicts and root boxes
    handles = (ctypes.c_void_p * max(len(mesh_names), 1))(*[dmeshes[nm].handle.value for nm in mesh_names])
    mc = np.ascontiguousarray(mat_color, np.float32).reshape(-1, 3)
    me = np.ascontiguousarray(mat_emissive, np.float32).reshape(-1, 3)
    h = ctypes.c_void_p()
    try:
        check(lib().rt_scene_compile(ctx.handle, len(mesh_names), handles, n_inst, srcs, n_sph, customs, ptr(mc),
                                     ptr(me), mc.shape[0], ctypes.byref(h)))
    except Exception:
        for name in mesh_names:
            dmeshes[name].finish()
        raise
    try:
        # the LBVH build is queued behind the flat-scene kernels before the verdicts are read
        # (a scene whose mesh fails is destroyed unbuilt-in-effect: nothing reads it)
        check(lib().rt_bvh_build(ctx.handle, h, QUALITIES[quality], None))
        for name in mesh_names:
            dmeshes[name].finish()
    except Exception:
        lib().rt_scene_destroy(h)
        raise
    for decl, m in inst_list:
        dm = dmeshes[decl.mesh]
        lo, hi = _corner_box(dm.bounds[:3], dm.bounds[3:], m)
        wlo.append(lo)
        whi.append(hi)
    for k, sph in enumerate(desc.spheres or ()):
        lo, hi, inv, llo, lhi, m = sph_boxes[k]
        placements.append((None, m, llo, lhi))
        wlo.append(lo)
        whi.append(hi)
        inverses.append(inv)
        inst_material.append(mat_index[sph.material])
    root_lo = np.min(np.array(wlo), axis=0)
    root_hi = np.max(np.array(whi), axis=0)
    n = sum(dmeshes[d.mesh].nf for d in desc.instances) + n_sph
    tlas = GpuTlas(ctx, h, n, QUALITIES[quality], np.array(sph_rows) if sph_rows else None,
                   n_instances=n_inst + n_sph, inverses=np.array(inverses), build=False)
    tlas.version = 1                                   # built above
    registry = IntersectorRegistry()
    if desc.spheres:
        registry.register(SPHERE_GEOM_TYPE, 0, sphere_intersector,
                          np.array([[*sph.center, sph.radius] for sph in desc.spheres]))
    lights = _light_rows(desc, mat_index, inst_list)
    if len(lights):
        rows = np.ascontiguousarray(np.concatenate([lights.v0, lights.v1, lights.v2, lights.normal, lights.emissive,
                                                    lights.area[:, None]], axis=1), np.float32)
        check(lib().rt_scene_set_lights(ctx.handle, tlas.handle, rows.shape[0], ptr(rows)))
    sc = Scene(camera=desc.camera, tlas=tlas, registry=registry, mat_color=mat_color, mat_emissive=mat_emissive,
               inst_material=np.array(inst_material, np.int64), lights=lights,
               sky=np.ascontiguousarray(desc.sky, np.float64), background=np.ascontiguousarray(desc.background,
                                                                                               np.float64),
               root_box_=(root_lo, root_hi))
    sc._placements = placements
    used = {d.mesh for d in desc.instances}
    sc._meshes = {name: dm for name, dm in dmeshes.items() if name in used}
    sc._light_src = (desc, mat_index, inst_list)
    return sc


def _corner_box(lo, hi, m):
    """World AABB of the 8 corners of a local box under a 3x4 matrix (accel.py:459-469)."""
    corners = np.array([[(lo, hi)[s & 1][0], (lo, hi)[(s >> 1) & 1][1], (lo, hi)[(s >> 2) & 1][2]]
                        for s in range(8)])
    pts = corners @ m[:, :3].T + m[:, 3]
    return pts.min(axis=0), pts.max(axis=0)


def _compile_two_level(desc, quality, device):
    """compile_scene through Blas / Instance / Tlas (scene.py:85-117), plus the device flatten."""
    from .twolevel import Blas, Instance, Tlas
    from .accel import sphere_aabbs
    if not desc.instances and not desc.spheres:
        raise BuildError("a scene needs at least one instance")
    mat_names = list(desc.materials)
    mat_index = {n: i for i, n in enumerate(mat_names)}
    mat_color = np.array([desc.materials[n].color for n in mat_names]).reshape(-1, 3)
    mat_emissive = np.array([desc.materials[n].emissive for n in mat_names]).reshape(-1, 3)
    blases, blas_of_mesh, instances, inst_material, inst_list = [], {}, [], [], []
    for name, mesh in desc.meshes.items():
        blas_of_mesh[name] = len(blases)
        blases.append(Blas.from_mesh(mesh.vertices, mesh.faces, quality, device=device))
    for decl in desc.instances:
        instances.append(Instance(blas_of_mesh[decl.mesh], decl.frame, decl.mask))
        inst_material.append(mat_index[decl.material])
        inst_list.append((decl, frame_to_matrix(decl.frame)))
    registry = IntersectorRegistry()
    if desc.spheres:
        rows = np.array([[*sph.center, sph.radius] for sph in desc.spheres], dtype=np.float64)
        registry.register(SPHERE_GEOM_TYPE, 0, sphere_intersector, sphere_data(rows))
        for i, sph in enumerate(desc.spheres):
            instances.append(Instance(len(blases), sph.frame, sph.mask))
            blases.append(Blas.from_aabbs(sphere_aabbs(rows[i:i + 1]), SPHERE_GEOM_TYPE, quality, data_offset=i,
                                          device=device))
            inst_material.append(mat_index[sph.material])
    tlas = Tlas(instances, blases, quality)
    flat = tlas.flatten(np.array(inst_material, np.int32), mat_color, mat_emissive, registry, QUALITIES[quality])
    lights = _light_rows(desc, mat_index, inst_list)
    if len(lights):
        rows = np.ascontiguousarray(np.concatenate([lights.v0, lights.v1, lights.v2, lights.normal, lights.emissive,
                                                    lights.area[:, None]], axis=1), np.float32)
        check(lib().rt_scene_set_lights(flat.ctx.handle, flat.handle, rows.shape[0], ptr(rows)))
    return Scene(camera=desc.camera, tlas=tlas, registry=registry, mat_color=mat_color, mat_emissive=mat_emissive,
                 inst_material=np.array(inst_material, np.int64), lights=lights,
                 sky=np.ascontiguousarray(desc.sky, np.float64),
                 background=np.ascontiguousarray(desc.background, np.float64), root_box_=tlas.root_box,
                 render_tlas=flat, _render_gen=tlas.generation, _render_bits=QUALITIES[quality])
