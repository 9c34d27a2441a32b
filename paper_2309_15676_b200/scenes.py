"""F1: path-traced gradient samplers for the BASELINE scenes (configs[0]
textured quad, [2] helix of spheres, [3]/[4] textured triangle meshes) and
their optimisation loops."""
from __future__ import annotations

import ctypes as C
import dataclasses  # noqa: F401
import math  # noqa: F401
from typing import Dict, List, Optional  # noqa: F401

import numpy as np
import torch

from . import _abi
from ._lib import DomainError, InvalidArgument, LogicError, MgError, check, load  # noqa: F401
from ._core import Context, Rng, _dtype_code, _p  # noqa: F401
from .estimators import FusedAdamUpdate, FusedMetaUpdate, GradientSamplePair  # noqa: F401


# ------------------------------------------------- F1 slice: textured quad
class QuadTextureProblem:
    """BASELINE.json configs[0] ("PR1 ref"): W x H image of one textured quad
    lit by one rectangular area light, direct lighting only, Lambertian BSDF;
    the parameters are an R x R RGB albedo texture ([3][R*R], channel-major).
    The reference has no renderer; scene and estimators are this
    repo's own, restated in oracle/metagrad_oracle.c.

    Textures: Rng(mix64(seed)).uniform() x 3R^2 (init seed 0, target seed 1,
    as the mini-render construction draws, problems.cpp:168-172); the target
    image is a target_spp-sample render of the target texture."""

    STREAM_TARGET = 7
    ITERATION_OFFSET = True  # the sampler honours mg_ctx_set_iteration_offset

    def __init__(self, width: int = 64, height: int = 64, tex_res: int = 32,
                 light=(8.0, 7.0, 6.0), init_seed: int = 0, target_seed: int = 1,
                 target_spp: int = 1024, dtype=torch.float64, ctx=None):
        self.ctx = ctx or Context.default()
        self.W, self.H, self.R, self.dtype = width, height, tex_res, dtype
        self.Le = (C.c_double * 3)(*light)
        n = 3 * tex_res * tex_res
        L = load()
        self.init = Rng([L.mg_mix64(init_seed)], ctx=self.ctx).uniform(n)[0].to(dtype)
        self.target_tex = Rng([L.mg_mix64(target_seed)], ctx=self.ctx).uniform(n)[0].to(dtype)
        self.target_img = torch.empty(3 * width * height, dtype=dtype, device="cuda")
        check(L.mg_quad_render(self.ctx.h, _dtype_code(self.target_tex), width, height, tex_res,
                               self.Le, target_spp, L.mg_mix64(target_seed), self.STREAM_TARGET,
                               _p(self.target_tex), _p(self.target_img)))
        self.accum = torch.zeros(6 * tex_res * tex_res, dtype=torch.int64, device="cuda")
        self.loss_buf = torch.zeros(1, dtype=torch.float64, device="cuda")

    def dim(self) -> int:
        return 3 * self.R * self.R

    def draws_per_sample(self) -> int:
        """Path samples per iteration: 2 proportional + 1 finite-difference spp."""
        return 3 * self.W * self.H

    def initial_params(self):
        return self.init.clone()

    def truth_params(self):
        return self.target_tex

    def render(self, tex, spp: int, key: int, stream: int = 3):
        img = torch.empty(3 * self.W * self.H, dtype=tex.dtype, device="cuda")
        check(load().mg_quad_render(self.ctx.h, _dtype_code(tex), self.W, self.H, self.R,
                                    self.Le, spp, key, stream, _p(tex.contiguous()), _p(img)))
        return img

    def sample_pair(self, now, prev, iteration: int, key: int, stream: int = 0, rows=None):
        """One gradient sample pair (prop, diff) for the L2 image loss; the
        returned pair's step_sq_norm is left to the fused update (device).
        rows=(r0, r1) restricts it to an image tile (partials of disjoint
        tiles sum exactly to the full pair)."""
        r0, r1 = rows if rows is not None else (0, self.H)
        prop, diff = torch.empty_like(now), torch.empty_like(now)
        check(load().mg_quad_sample_pair(self.ctx.h, _dtype_code(now), self.W, self.H, self.R,
                                         self.Le, _p(self.target_img), _p(now.contiguous()),
                                         _p(prev.contiguous()), key, iteration, stream, r0, r1,
                                         _p(self.accum), _p(prop), _p(diff), _p(self.loss_buf)))
        return GradientSamplePair(prop, diff)


class QuadTextureRun:
    """configs[0] optimisation loop on the device: per iteration one
    gradient-sample-pair launch (render + adjoint scatter) and one fused
    update (meta-estimator, or the Adam baseline), projection max(p, 0)."""

    def __init__(self, problem: QuadTextureProblem, optimizer: str = "meta", lr: float = 0.01,
                 seed: int = 0, replicate: int = 0, **kw):
        self.p = problem
        self.params = problem.initial_params()
        self.prev = self.params.clone()
        self.key = int(load().mg_stream_seed(seed, replicate))
        n = problem.dim()
        if optimizer == "meta":
            self.upd = FusedMetaUpdate(n, dtype=problem.dtype, lr=lr, project_lo=0.0,
                                       ctx=problem.ctx, **kw)
        elif optimizer == "adam":
            self.upd = FusedAdamUpdate(n, dtype=problem.dtype, lr=lr, project_lo=0.0,
                                       ctx=problem.ctx, **kw)
        else:
            raise InvalidArgument(_abi.MG_EINVAL, "optimizer must be meta or adam")
        self.optimizer = optimizer
        self.t = 0

    def step(self):
        pair = self.p.sample_pair(self.params, self.prev if self.optimizer == "meta" else
                                  self.params, self.t, self.key)
        new = self.prev  # ping-pong: pi_{t-1} buffer receives pi_{t+1}
        if self.optimizer == "meta":
            self.upd.step(pair.prop, pair.diff, self.params, new)
        else:
            self.upd.step(pair.prop, self.params, new)
        self.prev, self.params = self.params, new
        self.t += 1
        return pair

    def _step_at(self, iteration: int):
        pair = self.p.sample_pair(self.params, self.prev if self.optimizer == "meta" else
                                  self.params, iteration, self.key)
        new = self.prev
        if self.optimizer == "meta":
            self.upd.step(pair.prop, pair.diff, self.params, new)
        else:
            self.upd.step(pair.prop, self.params, new)
        self.prev, self.params = self.params, new

    def run(self, iterations: int, graph: bool = False):
        """`iterations` steps.  graph=True (meta optimiser): after the first
        (eager) step, a block of two steps — one ping-pong period — is
        captured once as a CUDA graph and replayed.  Nothing in a captured
        step comes from the host: the Philox iteration index is a device
        counter (mg_ctx_set_iteration_offset, advanced by the graph's last
        node) and the Moment2(beta_f) coefficient is formed on the device
        (prop_coef_device), so the replayed steps are the eager steps bit for
        bit.  Needs problem.ctx on a capturable (non-default) stream."""
        if not graph:
            for _ in range(iterations):
                self.step()
            return
        if self.optimizer != "meta":
            raise InvalidArgument(_abi.MG_EINVAL, "graph runs need the meta optimiser")
        if not getattr(self.p, "ITERATION_OFFSET", False):
            raise InvalidArgument(_abi.MG_EINVAL, "this problem's sampler has no device "
                                  "iteration offset; graph runs are unavailable")
        ctx = self.p.ctx
        if ctx.stream.cuda_stream == 0:
            raise InvalidArgument(_abi.MG_EINVAL, "graph runs need a context on a non-default stream")
        done = 0
        with torch.cuda.stream(ctx.stream):  # replays launch on the current stream
            while self.t < 1 and done < iterations:  # the first step initialises the state
                self.step()
                done += 1
            left = iterations - done
            if left >= 2:
                g = getattr(self, "_graph", None)
                if g is None:
                    g = self._capture()
                # the graph's buffer roles are fixed at capture: it expects
                # pi_t in the buffer that was `params` then.  After an odd
                # number of eager steps the roles are swapped; one eager step
                # realigns them
                if self.params.data_ptr() != self._graph_params_ptr:
                    self.step()
                    left -= 1
                self._it_dev.fill_(self.t)
                for _ in range(left // 2):
                    g.replay()
                    for _ in range(2):  # the host mirror of what the replay advanced
                        self.upd.t += 1
                        self.upd.beta_f_pow *= self.upd.beta_f
                    self.t += 2
                left %= 2
            for _ in range(left):
                self.step()

    def _capture(self):
        ctx, L = self.p.ctx, load()
        self._it_dev = torch.zeros(1, dtype=torch.int32, device="cuda")
        saved = (self.upd.t, self.upd.beta_f_pow, self.upd.device_coef)
        self.upd.device_coef = True
        g = torch.cuda.CUDAGraph()
        check(L.mg_ctx_set_iteration_offset(ctx.h, _p(self._it_dev)))
        try:
            with torch.cuda.graph(g, stream=ctx.stream):
                self._step_at(0)
                self._step_at(1)
                check(L.mg_iteration_offset_add(ctx.h, _p(self._it_dev), 2))
        finally:
            check(L.mg_ctx_set_iteration_offset(ctx.h, None))
            self.upd.t, self.upd.beta_f_pow, _ = saved
        self._graph = g
        self._graph_params_ptr = self.params.data_ptr()
        return g

    def loss_estimate(self) -> float:
        return float(self.p.loss_buf[0])

    def texture_error(self) -> float:
        return float(torch.linalg.vector_norm((self.params - self.p.target_tex).double()))


def helix_spheres(n: int = 64, radius: float = 0.1, turns: float = 4.0, helix_radius: float = 1.0,
                  y0: float = 0.3, y1: float = 2.3) -> np.ndarray:
    """configs[2] geometry: n spheres evenly along a helix (host libm
    cos/sin, computed once and shared by the device and the oracle)."""
    out = np.empty((n, 4))
    for k in range(n):
        phi = 2.0 * math.pi * turns * k / n
        out[k] = (helix_radius * math.cos(phi), y0 + (y1 - y0) * k / max(n - 1, 1),
                  helix_radius * math.sin(phi), radius)
    return out


class HelixProblem:
    """BASELINE.json configs[2]: a W x H render of a procedural helix of 64
    spheres (radius 0.1, 4 turns) on a diffuse ground plane under one area
    light plus a constant environment, depth-4 path tracing with NEE; the
    spheres' principled BSDF has 5 global parameters theta = (base r, g, b,
    metalness, roughness), initialised U(0,1) from seed 0 against seeded
    target values (seed 1).  Own renderer (oracle
    mgo_helix_*)."""

    ITERATION_OFFSET = True  # the sampler honours mg_ctx_set_iteration_offset

    def __init__(self, width: int = 256, height: int = 256, light=(10.0, 10.0, 10.0),
                 env=(0.2, 0.2, 0.2), ground=(0.5, 0.5, 0.5), init_seed: int = 0,
                 target_seed: int = 1, target_spp: int = 64, dtype=torch.float64, ctx=None):
        self.ctx = ctx or Context.default()
        self.W, self.H, self.dtype = width, height, dtype
        self.spheres_host = helix_spheres()
        self.spheres = torch.tensor(self.spheres_host, dtype=torch.float64, device="cuda")
        self.Le = (C.c_double * 3)(*light)
        self.env = (C.c_double * 3)(*env)
        self.ground = (C.c_double * 3)(*ground)
        L = load()
        self.init = Rng([L.mg_mix64(init_seed)], ctx=self.ctx).uniform(5)[0].to(dtype)
        tt = Rng([L.mg_mix64(target_seed)], ctx=self.ctx).uniform(5)[0]
        tt[4] = 0.3 + 0.7 * tt[4]  # target roughness in [0.3, 1] (well-conditioned highlights)
        self.target_theta = tt.to(dtype)
        self.target_img = self.render(self.target_theta, target_spp, int(L.mg_mix64(target_seed)))
        self.accum = torch.zeros(10, dtype=torch.int64, device="cuda")
        self.loss_buf = torch.zeros(1, dtype=torch.float64, device="cuda")

    def dim(self) -> int:
        return 5

    def draws_per_sample(self) -> int:
        """Paths per iteration: 2 proportional + 1 finite-difference spp."""
        return 3 * self.W * self.H

    def initial_params(self):
        return self.init.clone()

    def render(self, theta, spp: int, key: int):
        img = torch.empty(3 * self.W * self.H, dtype=theta.dtype, device="cuda")
        check(load().mg_helix_render(self.ctx.h, _dtype_code(theta), self.W, self.H,
                                     self.spheres.shape[0], _p(self.spheres), self.Le, self.env,
                                     self.ground, _p(theta.contiguous()), spp, key, _p(img)))
        return img

    def sample_pair(self, now, prev, iteration: int, key: int, rows=None):
        r0, r1 = rows if rows is not None else (0, self.H)
        prop, diff = torch.empty_like(now), torch.empty_like(now)
        check(load().mg_helix_sample_pair(
            self.ctx.h, _dtype_code(now), self.W, self.H, self.spheres.shape[0], _p(self.spheres),
            self.Le, self.env, self.ground, _p(self.target_img), _p(now.contiguous()),
            _p(prev.contiguous()), key, iteration, r0, r1, _p(self.accum), _p(prop), _p(diff),
            _p(self.loss_buf)))
        return GradientSamplePair(prop, diff)


class HelixRun(QuadTextureRun):
    """configs[2] optimisation loop (same structure as QuadTextureRun); the 5
    parameters (colours, metalness, roughness) are projected to [0, 1]."""

    def __init__(self, problem, optimizer: str = "meta", lr: float = 0.01, seed: int = 0,
                 replicate: int = 0, **kw):
        if optimizer == "meta":
            kw.setdefault("project_hi", 1.0)
        super().__init__(problem, optimizer, lr, seed, replicate, **kw)


# ------------------------------------- F1 slice 3: textured mesh scene
MESH_VIEW_LAYOUT = ("cam[3] fwd[3] right[3] up[3] tan_half_fov light_y light_x0 light_x1 "
                    "light_z0 light_z1 Le[3] env[3] max_vertices")


def _sphere_triangles(center, radius_fn, n_theta: int, n_phi: int):
    """UV-sphere tessellation: (v0, v1, v2, uv0, uv1, uv2) lists; single
    triangles at the poles (no degenerate ones).  uv = (phi/2pi, theta/pi)."""
    th = np.pi * np.arange(n_theta + 1) / n_theta
    ph = 2.0 * np.pi * np.arange(n_phi + 1) / n_phi
    T_, P_ = np.meshgrid(th, ph, indexing="ij")
    rad = radius_fn(T_, P_)
    pos = np.stack([center[0] + rad * np.sin(T_) * np.cos(P_), center[1] + rad * np.cos(T_),
                    center[2] + rad * np.sin(T_) * np.sin(P_)], axis=-1)
    uv = np.stack([P_ / (2.0 * np.pi), T_ / np.pi], axis=-1)
    # per grid cell (row-major): (a, b, d) unless in the first row, then
    # (a, d, c) unless in the last row; a = (i, j), b = (i, j+1),
    # c = (i+1, j), d = (i+1, j+1)
    I, J = np.meshgrid(np.arange(n_theta), np.arange(n_phi), indexing="ij")
    I, J = I.reshape(-1), J.reshape(-1)
    ti = np.stack([np.stack([I, I, I + 1], 1), np.stack([I, I + 1, I + 1], 1)], 1)
    tj = np.stack([np.stack([J, J + 1, J + 1], 1), np.stack([J, J + 1, J], 1)], 1)
    keep = np.stack([I != 0, I != n_theta - 1], 1).reshape(-1)
    ti, tj = ti.reshape(-1, 3)[keep], tj.reshape(-1, 3)[keep]
    return pos[ti, tj], uv[ti, tj]


def mesh_scene_geometry(sphere_res=(24, 48), displaced_res=(100, 100), seed: int = 3,
                        displacement: float = 0.12):
    """BASELINE.json configs[3] geometry (seed-generated):
    object 0 a ground quad (y = 0, x, z in [-2.5, 2.5]), object 1 a sphere
    (centre (-0.9, 0.5, 0), radius 0.5), object 2 a seeded displaced sphere
    (centre (0.8, 0.55, 0.1), radius 0.5 (1 + displacement * noise),
    ~2 * n_theta * n_phi triangles: 19.8k at the default 100 x 100).
    Returns (records [T][18] fp64, object ids [T] int32, nobj)."""
    quad_v = np.array([[[-2.5, 0.0, -2.5], [2.5, 0.0, -2.5], [2.5, 0.0, 2.5]],
                       [[-2.5, 0.0, -2.5], [2.5, 0.0, 2.5], [-2.5, 0.0, 2.5]]])
    quad_w = (quad_v[:, :, [0, 2]] + 2.5) / 5.0
    sph_v, sph_w = _sphere_triangles((-0.9, 0.5, 0.0), lambda t, p: 0.5 + 0.0 * t, *sphere_res)
    rs = np.random.RandomState(seed)
    waves = [(rs.uniform(-1, 1), rs.randint(1, 6), rs.randint(1, 7), rs.uniform(0, 2 * np.pi))
             for _ in range(6)]

    def disp(t, p):
        noise = sum(a * np.sin(m * t) * np.cos(g * p + q) for a, m, g, q in waves) / len(waves)
        return 0.5 * (1.0 + displacement * noise * 2.0)
    dsp_v, dsp_w = _sphere_triangles((0.8, 0.55, 0.1), disp, *displaced_res)
    V = np.concatenate([quad_v, sph_v, dsp_v])
    Wuv = np.concatenate([quad_w, sph_w, dsp_w])
    obj = np.concatenate([np.zeros(len(quad_v)), np.ones(len(sph_v)),
                          np.full(len(dsp_v), 2)]).astype(np.int32)
    e1 = V[:, 1] - V[:, 0]
    e2 = V[:, 2] - V[:, 0]
    n = np.cross(e1, e2)
    n = n / np.linalg.norm(n, axis=1, keepdims=True)
    rec = np.concatenate([V[:, 0], e1, e2, n, Wuv[:, 0], Wuv[:, 1] - Wuv[:, 0],
                          Wuv[:, 2] - Wuv[:, 0]], axis=1)
    return np.ascontiguousarray(rec), obj, 3


def mesh_large_scene_geometry(n_spheres: int = 15, res=(130, 130), seed: int = 5,
                              displacement: float = 0.15):
    """BASELINE.json configs[4] geometry: object 0 a ground quad, objects
    1..n_spheres seeded displaced spheres (radius 0.35) on a 5-wide grid —
    16 objects and ~502k triangles at the default 130 x 130 tessellation."""
    quad_v = np.array([[[-3.0, 0.0, -2.5], [3.0, 0.0, -2.5], [3.0, 0.0, 2.5]],
                       [[-3.0, 0.0, -2.5], [3.0, 0.0, 2.5], [-3.0, 0.0, 2.5]]])
    quad_w = np.stack([(quad_v[:, :, 0] + 3.0) / 6.0, (quad_v[:, :, 2] + 2.5) / 5.0], axis=-1)
    rs = np.random.RandomState(seed)
    Vs, Ws, objs = [quad_v], [quad_w], [np.zeros(2)]
    for k in range(n_spheres):
        cx = -2.0 + 1.0 * (k % 5) + rs.uniform(-0.1, 0.1)
        cz = -1.2 + 1.0 * (k // 5) + rs.uniform(-0.1, 0.1)
        waves = [(rs.uniform(-1, 1), rs.randint(1, 6), rs.randint(1, 7), rs.uniform(0, 2 * np.pi))
                 for _ in range(5)]

        def rad(t, p, waves=waves):
            noise = sum(a * np.sin(m * t) * np.cos(g * p + q) for a, m, g, q in waves) / len(waves)
            return 0.35 * (1.0 + displacement * noise * 2.0)
        v, w = _sphere_triangles((cx, 0.4, cz), rad, *res)
        Vs.append(v)
        Ws.append(w)
        objs.append(np.full(len(v), k + 1))
    V, Wuv = np.concatenate(Vs), np.concatenate(Ws)
    obj = np.concatenate(objs).astype(np.int32)
    e1 = V[:, 1] - V[:, 0]
    e2 = V[:, 2] - V[:, 0]
    n = np.cross(e1, e2)
    n = n / np.linalg.norm(n, axis=1, keepdims=True)
    rec = np.concatenate([V[:, 0], e1, e2, n, Wuv[:, 0], Wuv[:, 1] - Wuv[:, 0],
                          Wuv[:, 2] - Wuv[:, 0]], axis=1)
    return np.ascontiguousarray(rec), obj, n_spheres + 1


def mesh_scene_view(max_vertices: int = 6, light=(6.0, 6.0, 6.0), env=(0.25, 0.3, 0.35),
                    cam=(0.0, 1.6, 4.5), look_at=(0.0, 0.45, 0.0), tan_half_fov: float = 0.45,
                    light_y: float = 3.0, light_rect=(-1.0, 1.0, -1.0, 1.0)):
    """view[25] (layout MESH_VIEW_LAYOUT): pinhole camera, rectangular light
    at y = light_y over x in [x0, x1], z in [z0, z1] facing down, constant
    environment."""
    cam = np.asarray(cam, dtype=np.float64)
    fwd = np.asarray(look_at, dtype=np.float64) - cam
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, [0.0, 1.0, 0.0])
    right /= np.linalg.norm(right)
    up = np.cross(right, fwd)
    return np.concatenate([cam, fwd, right, up, [tan_half_fov, light_y, *light_rect],
                           light, env, [float(max_vertices)]]).astype(np.float64)


def smooth_noise_textures(nobj: int, R: int, seed: int, grid: int = 6,
                          base_range=(0.15, 0.85), rough_range=(0.25, 0.9), channels: int = 4,
                          metal_range=(0.0, 0.6)) -> np.ndarray:
    """Seeded smooth-noise textures [nobj][channels][R*R] (bilinear upsampling
    of a grid x grid lattice of uniforms): base colour, roughness and (5
    channels) metalness."""
    rs = np.random.RandomState(seed)
    x = (np.arange(R) + 0.5) / R * (grid - 1)
    i0 = np.minimum(x.astype(int), grid - 2)
    f = x - i0
    out = np.empty((nobj, channels, R * R))
    for o in range(nobj):
        for c in range(channels):
            g = rs.uniform(0, 1, (grid, grid))
            rows = g[i0] * (1 - f)[:, None] + g[i0 + 1] * f[:, None]
            img = rows[:, i0] * (1 - f)[None, :] + rows[:, i0 + 1] * f[None, :]
            lo, hi = base_range if c < 3 else (rough_range if c == 3 else metal_range)
            out[o, c] = (lo + (hi - lo) * img).reshape(-1)
    return out


class MeshScene:
    """A triangle scene on the device (BVH built on the host, mg_meshscene_*)."""

    def __init__(self, records: np.ndarray, obj: np.ndarray, nobj: int, tex_res: int, view,
                 ctx=None, channels: int = 4):
        self.ctx = ctx or Context.default()
        self.records = np.ascontiguousarray(records, dtype=np.float64)
        self.obj = np.ascontiguousarray(obj, dtype=np.int32)
        self.nobj, self.R, self.channels = nobj, tex_res, channels
        self.view = np.ascontiguousarray(view, dtype=np.float64)
        h = C.c_void_p()
        check(load().mg_meshscene_create(self.ctx.h, self.records.shape[0],
                                         self.records.ctypes.data_as(C.c_void_p),
                                         self.obj.ctypes.data_as(C.c_void_p), nobj, tex_res,
                                         channels, C.byref(h)))
        self.h = h

    def info(self):
        nodes, depth, params = C.c_int32(), C.c_int32(), C.c_int64()
        check(load().mg_meshscene_info(self.h, C.byref(nodes), C.byref(depth), C.byref(params)))
        return {"nodes": nodes.value, "depth": depth.value, "params": params.value,
                "triangles": self.records.shape[0]}

    def params(self) -> int:
        return self.nobj * self.channels * self.R * self.R

    def intersect(self, rays: torch.Tensor):
        """rays: CUDA fp64 [n][6] -> (t [n], triangle [n])"""
        n = rays.shape[0]
        t = torch.empty(n, dtype=torch.float64, device=rays.device)
        k = torch.empty(n, dtype=torch.int32, device=rays.device)
        check(load().mg_meshscene_intersect(self.ctx.h, self.h, n, _p(rays.contiguous()), _p(t),
                                            _p(k)))
        return t, k

    def render(self, theta, W: int, H: int, spp: int, key: int):
        img = torch.empty(3 * W * H, dtype=theta.dtype, device="cuda")
        check(load().mg_meshscene_render(self.ctx.h, self.h, _dtype_code(theta), W, H,
                                         self.view.ctypes.data_as(C.c_void_p), spp, key,
                                         _p(theta.contiguous()), _p(img)))
        return img

    def __del__(self):
        try:
            if getattr(self, "h", None):
                load().mg_meshscene_destroy(self.h)
        except Exception:
            pass


class MeshTextureProblem:
    """BASELINE.json configs[3]: W x H render of the 3-object mesh scene,
    each object with an R x R RGB albedo + roughness texture (3 * 4 * R^2
    parameters, ~3.1M at R = 512), targets seeded smooth noise (seed 1),
    initialised to base 0.5 / roughness 0.5, depth-6 NEE path tracing,
    1 FD + 2 proportional spp (paths A, B, C).  Own renderer (DESIGN.md §12,
    oracle mgo_mesh_*)."""

    ITERATION_OFFSET = True  # the sampler honours mg_ctx_set_iteration_offset

    def __init__(self, width: int = 512, height: int = 512, tex_res: int = 512,
                 sphere_res=(24, 48), displaced_res=(100, 100), max_vertices: int = 6,
                 target_seed: int = 1, target_spp: int = 16, dtype=torch.float32, ctx=None,
                 channels: int = 4, prop_paths: int = 2, geometry=None, view=None):
        self.ctx = ctx or Context.default()
        self.W, self.H, self.R, self.dtype = width, height, tex_res, dtype
        self.channels, self.prop_paths = channels, prop_paths
        rec, obj, nobj = geometry if geometry is not None else \
            mesh_scene_geometry(sphere_res, displaced_res)
        view = view if view is not None else mesh_scene_view(max_vertices)
        self.scene = MeshScene(rec, obj, nobj, tex_res, view, self.ctx, channels)
        n = self.scene.params()
        self.target_tex = torch.tensor(
            smooth_noise_textures(nobj, tex_res, target_seed, channels=channels).reshape(-1),
            device="cuda").to(dtype)
        init = np.full((nobj, channels, tex_res * tex_res), 0.5)
        if channels == 5:
            init[:, 4] = 0.1
        self.init = torch.tensor(init.reshape(-1), device="cuda").to(dtype)
        self.target_img = self.scene.render(self.target_tex, width, height, target_spp,
                                            int(load().mg_mix64(target_seed)))
        self.accum = torch.zeros(2 * n, dtype=torch.int64, device="cuda")
        self.touch = None
        self.loss_buf = torch.zeros(1, dtype=torch.float64, device="cuda")

    def dim(self) -> int:
        return self.scene.params()

    def enable_touch_map(self, enable: bool = True):
        """One bit per texel cell of self.accum, set by sample_pair(...,
        finalize=False) for every cell it adds to and consumed by
        FusedMetaUpdate.step_fixed(..., touch=self.touch)
        (mg_meshscene_set_touch_map / mg_meta_update_fixed_touch)."""
        if enable and self.touch is None:
            cells = self.dim() // self.scene.channels
            # set conservatively: accum may already hold a pair
            self.touch = torch.full(((cells + 31) // 32,), -1, dtype=torch.int32, device="cuda")
        elif not enable:
            self.touch = None
        check(load().mg_meshscene_set_touch_map(self.scene.h, _p(self.touch)))
        return self.touch

    def draws_per_sample(self) -> int:
        """Paths per iteration: prop_paths proportional + 1 finite-difference spp."""
        return (self.prop_paths + 1) * self.W * self.H

    def initial_params(self):
        return self.init.clone()

    def sample_pair(self, now, prev, iteration: int, key: int, rows=None, finalize: bool = True):
        """finalize=False: the pair stays in self.accum (texel-interleaved
        fixed point) for FusedMetaUpdate.step_fixed; returns None."""
        r0, r1 = rows if rows is not None else (0, self.H)
        prop, diff = (torch.empty_like(now), torch.empty_like(now)) if finalize else (None, None)
        check(load().mg_meshscene_sample_pair(
            self.ctx.h, self.scene.h, _dtype_code(now), self.W, self.H,
            self.scene.view.ctypes.data_as(C.c_void_p), _p(self.target_img), _p(now.contiguous()),
            _p(prev.contiguous()), key, iteration, r0, r1, self.prop_paths, _p(self.accum),
            _p(prop), _p(diff), _p(self.loss_buf)))
        return GradientSamplePair(prop, diff) if finalize else None

    def fixed_layout(self):
        """(cells, channels, texels per object) of self.accum's pair."""
        R2 = self.scene.R * self.scene.R
        return self.dim() // self.scene.channels, self.scene.channels, R2


    def sample_pair_sharded(self, now, prev, iteration: int, key: int, rows, acc_ptrs,
                            shard: int):
        """Rows `rows` of the image, contributions atomically added into the
        owning ranks' fixed-point accumulators (acc_ptrs[r]: device int64
        [2][shard], e.g. symmetric-memory peer pointers): the adjoint
        scatter and the reduce-scatter of a tile-sharded step in one kernel
        (mg_meshscene_sample_pair_sharded).  Loss of the rows -> loss_buf."""
        ptrs = (C.c_void_p * len(acc_ptrs))(*[int(x) for x in acc_ptrs])
        check(load().mg_meshscene_sample_pair_sharded(
            self.ctx.h, self.scene.h, _dtype_code(now), self.W, self.H,
            self.scene.view.ctypes.data_as(C.c_void_p), _p(self.target_img), _p(now.contiguous()),
            _p(prev.contiguous()), key, iteration, rows[0], rows[1], self.prop_paths,
            len(acc_ptrs), ptrs, shard, _p(self.loss_buf)))


def fixed_finalize(accum, prop, diff, ctx=None):
    """accum (int64 [2][n], 2^-40 units) -> prop, diff; accum zeroed."""
    ctx = ctx or Context.default()
    check(load().mg_fixed_finalize(ctx.h, _dtype_code(prop), prop.numel(), _p(accum), _p(prop),
                                   _p(diff)))


def large_scene_view(max_vertices: int = 8):
    """configs[4] camera/light over the 5 x 3 grid of objects."""
    return mesh_scene_view(max_vertices, light=(8.0, 8.0, 8.0), cam=(0.0, 2.8, 4.4),
                           look_at=(0.0, 0.2, -0.3), tan_half_fov=0.55, light_y=3.5,
                           light_rect=(-1.5, 1.5, -1.5, 1.0))


class MeshLargeProblem(MeshTextureProblem):
    """BASELINE.json configs[4]: 1024 x 1024 image, 16 objects (ground quad +
    15 seeded displaced spheres, ~502k triangles), each with a 1024 x 1024
    texture of base r, g, b, roughness and metalness (16 * 5 * 1024^2 =
    83.9M parameters), depth 8 with NEE, 1 FD + 4 proportional spp."""

    def __init__(self, width: int = 1024, height: int = 1024, tex_res: int = 1024,
                 res=(130, 130), max_vertices: int = 8, target_seed: int = 1,
                 target_spp: int = 4, dtype=torch.float32, ctx=None, prop_paths: int = 4):
        super().__init__(width, height, tex_res, max_vertices=max_vertices,
                         target_seed=target_seed, target_spp=target_spp, dtype=dtype, ctx=ctx,
                         channels=5, prop_paths=prop_paths,
                         geometry=mesh_large_scene_geometry(res=res),
                         view=large_scene_view(max_vertices))


class MeshTextureRun(QuadTextureRun):
    """configs[3] optimisation loop: sample pair + fused update per
    iteration; texture values projected to [0, 1] (meta)."""

    def __init__(self, problem, optimizer: str = "meta", lr: float = 0.01, seed: int = 0,
                 replicate: int = 0, fused: bool = True, touch_map: bool = True, **kw):
        if optimizer == "meta":
            kw.setdefault("project_hi", 1.0)
        super().__init__(problem, optimizer, lr, seed, replicate, **kw)
        # the loop ping-pongs its parameter buffers (prev at t+1 == now at t,
        # untouched in between): the scene may reuse prev's texel-major copy
        check(load().mg_meshscene_set_prev_reuse(problem.scene.h, 1))
        # meta optimiser: the update consumes the fixed-point accumulator
        # directly (mg_meta_update_fixed) — step() then returns None;
        # fused=False keeps the planar pair (step() returns it)
        self.fused = bool(fused) and optimizer == "meta"
        # ... and reads / zeroes only the accumulator cells a path reached
        if self.fused:
            problem.enable_touch_map(bool(touch_map))

    def step(self):
        if not self.fused:
            return super().step()
        self._step_at(self.t)
        self.t += 1
        return None

    def _step_at(self, iteration: int):
        if not self.fused:
            return super()._step_at(iteration)
        self.p.sample_pair(self.params, self.prev, iteration, self.key, finalize=False)
        new = self.prev
        cells, nch, r2 = self.p.fixed_layout()
        self.upd.step_fixed(self.p.accum, cells, nch, r2, self.params, new, touch=self.p.touch)
        self.prev, self.params = self.params, new
