"""B200-native ray tracer: the reference ``pathtrace`` API over sm_100a CUDA kernels.

Public surface mirrors the reference package (pkg/src/pathtrace/__init__.py)
for the hot path: scene load -> ``compile_scene`` (GPU LBVH) ->
``closest_hit_batch`` / ``render_frame``.  Everything heavy runs in
librt_b200.so (built by ``__graft_entry__.build()``); there is no CPU fallback.
"""

from .camera import Camera, CameraError, pixel_to_uv
from .frames import FULL_MASK, SrtFrame, frame_to_matrix, invert_affine
from .scene_io import (AccumBuffer, InstanceDecl, Material, ParseError, SceneDescription, TriangleMesh,
                       load_obj, load_scene, parse_obj, parse_scene, ppm_bytes, resolve, write_ppm)
from ._native import BuildError, RegistryError
from .scene import Scene, compile_scene
from .accel import (CUSTOM, SPHERE_GEOM_TYPE, TRIANGLES, IntersectorRegistry, any_hit_batch, closest_hit_batch,
                    make_sphere_registry, sphere_aabbs, sphere_data, sphere_intersector, trace_any, trace_closest)
from .integrators import INTEGRATORS, IntegratorConfig, render_frame, render_into
from .twolevel import Blas, Instance, Tlas, build_tlas, transform_ray_to_local

__version__ = "0.1.0"
