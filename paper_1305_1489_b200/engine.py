"""Reference-shaped Python API over the C ABI (device memory held in torch tensors).

The names mirror the reference library (proj/include/hdg/*.hpp): `geometry`,
`build_condense` (= build_element_matrices -> local_blocks -> condense),
`recover` (= gather_traces + local_recover), `assemble`, `postprocess_star`,
`convection_bilinear_matrices`, `element_matrices`. Layouts follow the
reference: a Batch3 r x c x n is returned as an (n, r, c) view of the
column-major slices, an r x Nelt matrix as an (Nelt, r) view (column K contiguous).
torch provides device memory and the stream; all compute runs in the CUDA
kernels of libhdg_b200.so (no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence, Union

import numpy as np
import torch

from . import _lib as L
from .fields import FieldProgram, compile_field


def dim3(k: int) -> int:
    return (k + 1) * (k + 2) * (k + 3) // 6


def dim2(k: int) -> int:
    return (k + 1) * (k + 2) // 2


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    raise TypeError(type(t))


# ------------------------------------------------------------------- fields
class Field:
    """A coefficient field: constant, program (expression) or device samples."""

    def __init__(self, kind: int, value: float = 0.0, samples: Optional[torch.Tensor] = None,
                 prog: Optional[FieldProgram] = None):
        self.kind, self.value, self.samples, self.prog = kind, float(value), samples, prog
        self._keep = []

    @staticmethod
    def const(v: float) -> "Field":
        return Field(L.FIELD_CONST, value=v)

    @staticmethod
    def program(expr: Union[str, FieldProgram]) -> "Field":
        prog = expr if isinstance(expr, FieldProgram) else compile_field(expr)
        return Field(L.FIELD_PROGRAM, prog=prog)

    @staticmethod
    def sampled(t: torch.Tensor) -> "Field":
        if t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
            raise ValueError("sampled fields must be contiguous float64 CUDA tensors (nq x nelt)")
        return Field(L.FIELD_SAMPLED, samples=t)

    def c_struct(self) -> L.hdg_field:
        f = L.hdg_field()
        f.kind = self.kind
        f.value = self.value
        if self.kind == L.FIELD_SAMPLED:
            f.samples = self.samples.data_ptr()
        elif self.kind == L.FIELD_PROGRAM:
            ops = (C.c_int * len(self.prog.ops))(*self.prog.ops)
            cs = (C.c_double * max(1, len(self.prog.consts)))(*self.prog.consts)
            self._keep = [ops, cs]
            f.ops = C.cast(ops, C.c_void_p)
            f.nops = len(self.prog.ops)
            f.consts = C.cast(cs, C.c_void_p)
            f.nconst = len(self.prog.consts)
        return f


def as_field(x) -> Field:
    if isinstance(x, Field):
        return x
    if isinstance(x, (int, float)):
        return Field.const(float(x))
    if isinstance(x, (str, FieldProgram)):
        return Field.program(x)
    if isinstance(x, torch.Tensor):
        return Field.sampled(x)
    raise TypeError(f"cannot make a field from {type(x)}")


# --------------------------------------------------------------------- mesh
class HostMesh:
    """Reference RawMesh + expand() numbering, held by the C++ host layer."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and L is not None and L.lib is not None:  # module teardown at exit
            L.lib().hdg_b200_mesh_free(h)
            self._h = None

    @classmethod
    def box(cls, nx: int, ny: Optional[int] = None, nz: Optional[int] = None,
            bc: str = "dirichlet_top_bottom", perturb: float = 0.0, seed: int = 1305,
            keep_plane_z: float = 0.5, expand: bool = True) -> "HostMesh":
        h = C.c_void_p()
        L.check(L.lib().hdg_b200_mesh_box(nx, ny or nx, nz or nx, L.BC[bc], perturb, seed, keep_plane_z,
                                          C.byref(h)))
        m = cls(h)
        if expand:
            m.expand()
        return m

    @classmethod
    def from_raw(cls, coords, elements, dirichlet, neumann, expand: bool = True) -> "HostMesh":
        co = np.asfortranarray(coords, dtype=np.float64)
        el = np.asfortranarray(elements, dtype=np.int32)
        di = np.asfortranarray(dirichlet, dtype=np.int32).reshape(-1, 3, order="F") if len(dirichlet) else np.zeros((0, 3), np.int32)
        ne = np.asfortranarray(neumann, dtype=np.int32).reshape(-1, 3, order="F") if len(neumann) else np.zeros((0, 3), np.int32)
        h = C.c_void_p()
        L.check(L.lib().hdg_b200_mesh_create(co.shape[0], co.ctypes.data, el.shape[0], el.ctypes.data,
                                             di.shape[0], di.ctypes.data if di.size else None,
                                             ne.shape[0], ne.ctypes.data if ne.size else None, C.byref(h)))
        m = cls(h)
        if expand:
            m.expand()
        return m

    def expand(self) -> None:
        L.check(L.lib().hdg_b200_mesh_expand(self._h))

    @property
    def dims(self):
        d = (C.c_int64 * 6)()
        L.check(L.lib().hdg_b200_mesh_dims(self._h, d))
        return dict(nver=d[0], nelt=d[1], nfc=d[2], ndir=d[3], nneu=d[4], expanded=bool(d[5]))

    def _get(self, what, shape, dtype):
        out = np.zeros(int(np.prod(shape)), dtype=dtype)
        if out.size:
            L.check(L.lib().hdg_b200_mesh_copy(self._h, what, out.ctypes.data))
        return out.reshape(shape, order="F")

    @property
    def n_elements(self): return self.dims["nelt"]

    @property
    def n_faces(self): return self.dims["nfc"]

    @property
    def coordinates(self): return self._get(L.MESH_COORDS, (self.dims["nver"], 3), np.float64)

    @property
    def elements(self): return self._get(L.MESH_ELEMENTS, (self.dims["nelt"], 4), np.int32)

    @property
    def dirichlet(self): return self._get(L.MESH_DIRICHLET, (self.dims["ndir"], 3), np.int32)

    @property
    def neumann(self): return self._get(L.MESH_NEUMANN, (self.dims["nneu"], 3), np.int32)

    @property
    def faces(self): return self._get(L.MESH_FACES, (self.dims["nfc"], 3), np.int32)

    @property
    def facetype(self): return self._get(L.MESH_FACETYPE, (self.dims["nfc"],), np.uint8)

    @property
    def facebyele(self): return self._get(L.MESH_FACEBYELE, (self.dims["nelt"], 4), np.int32)

    def pattern(self):
        """(facebase[nfc+1], nbr[nfc,8], slot[nelt,16]) of the skeleton sparsity."""
        tot = C.c_int64()
        L.check(L.lib().hdg_b200_pattern_dims(self._h, C.byref(tot)))
        d = self.dims
        fb = np.zeros(d["nfc"] + 1, np.int64)
        nb = np.zeros((d["nfc"], 8), np.int32)
        sl = np.zeros((d["nelt"], 16), np.uint8)
        L.check(L.lib().hdg_b200_pattern_build(self._h, fb.ctypes.data, nb.ctypes.data, sl.ctypes.data))
        return fb, nb, sl


@dataclass
class DeviceMesh:
    nver: int
    nelt: int
    nfc: int
    coords: torch.Tensor     # (3, nver) float64 == reference Nver x 3 column-major
    elements: torch.Tensor   # (4, nelt) int32
    faces: torch.Tensor      # (3, nfc) int32
    facebyele: torch.Tensor  # (4, nelt) int32
    facetype: torch.Tensor   # (nfc,) uint8
    ndir: int = 0            # Dirichlet faces are [0, ndir) (mesh.cpp:99-116)
    nneu: int = 0            # Neumann faces are [ndir, ndir + nneu)


@dataclass
class Geometry:
    volume: torch.Tensor  # (nelt,)
    piola: torch.Tensor   # (9, nelt)
    normals: torch.Tensor  # (12, nelt)
    perm: torch.Tensor    # (4, nelt) int32
    T: torch.Tensor       # (4, nelt)
    verts: torch.Tensor   # (12, nelt)
    area: torch.Tensor    # (nfc,)

    @property
    def nelt(self) -> int:
        return self.volume.numel()

    def c_struct(self) -> L.hdg_geometry:
        g = L.hdg_geometry()
        for n in ("volume", "piola", "normals", "perm", "T", "verts", "area"):
            setattr(g, n, getattr(self, n).data_ptr())
        return g


@dataclass
class CondensedSystem:
    C: torch.Tensor        # flat m*m*nelt (Batch3)
    Cf: torch.Tensor       # flat m*nelt
    factors: Optional[torch.Tensor]
    m: int

    def C_slices(self) -> torch.Tensor:
        """(nelt, m, m) with [K, i, j] = C_K(i, j)."""
        return self.C.view(-1, self.m, self.m).transpose(1, 2)

    def Cf_cols(self) -> torch.Tensor:
        """(nelt, m) with [K, i] = Cf(i, K)."""
        return self.Cf.view(-1, self.m)


@dataclass
class LocalSolution:
    qx: torch.Tensor  # (nelt, d3) == reference d3 x Nelt column-major
    qy: torch.Tensor
    qz: torch.Tensor
    u: torch.Tensor


@dataclass
class SkeletonSystem:
    rowptr: torch.Tensor  # int64 (ndof+1)
    colidx: torch.Tensor  # int32 (nnz)
    vals: torch.Tensor    # float64 (nnz)
    b: torch.Tensor       # float64 (ndof)
    d2: int


@dataclass
class DevicePattern:
    facebase: torch.Tensor  # int64 (nfc+1)
    nbr: torch.Tensor       # int32 (nfc, 8)
    slot: torch.Tensor      # uint8 (nelt, 16)
    rowptr: Optional[torch.Tensor] = None
    colidx: Optional[torch.Tensor] = None
    sides: Optional[torch.Tensor] = None  # int32 (nfc, 2): e*4+l of each face's elements (K4 by faces)


class Engine:
    """One device + stream + the reference-element tables of one degree."""

    def __init__(self, device: int = 0, stream: Optional[torch.cuda.Stream] = None):
        self.device = torch.device("cuda", device)
        self.stream = stream or torch.cuda.current_stream(self.device)
        self._ctx = C.c_void_p()
        L.check(L.lib().hdg_b200_create(device, C.c_void_p(self.stream.cuda_stream), C.byref(self._ctx)))
        self.k = None

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx and L is not None and L.lib is not None:  # module teardown at exit
            L.lib().hdg_b200_destroy(ctx)
            self._ctx = None

    # ---------------------------------------------------------------- setup
    def set_stream(self, stream: torch.cuda.Stream) -> None:
        self.stream = stream
        L.check(L.lib().hdg_b200_set_stream(self._ctx, C.c_void_p(stream.cuda_stream)))

    def set_degree(self, k: int, tet_deg: Optional[int] = None, tri_deg: Optional[int] = None) -> None:
        """study.cpp:13-15: tet_rule(2k+2), tri_rule(2k+2), build_tables(k)."""
        tet_deg = 2 * k + 2 if tet_deg is None else tet_deg
        tri_deg = 2 * k + 2 if tri_deg is None else tri_deg
        L.check(L.lib().hdg_b200_set_degree(self._ctx, k, tet_deg, tri_deg))
        self.k, self.tet_deg, self.tri_deg = k, tet_deg, tri_deg

    def set_postprocess_rule(self, tet_deg: Optional[int] = None) -> None:
        """study.cpp:33-34: tet_rule(2(k+1)+2), build_tables(k+1)."""
        tet_deg = 2 * (self.k + 1) + 2 if tet_deg is None else tet_deg
        L.check(L.lib().hdg_b200_set_postprocess_rule(self._ctx, tet_deg))

    @property
    def dims(self):
        d = (C.c_int64 * 8)()
        L.check(L.lib().hdg_b200_dims(self._ctx, d))
        return dict(k=d[0], d3=d[1], d2=d[2], nq=d[3], nqd=d[4], factors=d[5], nq_post=d[6], d3_post=d[7])

    def table(self, name: str) -> np.ndarray:
        out = np.zeros(1 << 20)
        L.check(L.lib().hdg_b200_copy_table(self._ctx, L.TABLES[name], out.ctypes.data, out.size))
        return out

    def upload(self, mesh: HostMesh) -> DeviceMesh:
        d = mesh.dims
        dev = self.device
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).to(dev, dt)
        return DeviceMesh(d["nver"], d["nelt"], d["nfc"], t(mesh.coordinates, torch.float64),
                          t(mesh.elements, torch.int32), t(mesh.faces, torch.int32),
                          t(mesh.facebyele, torch.int32),
                          torch.from_numpy(mesh.facetype).to(dev), d["ndir"], d["nneu"])

    def synchronize(self) -> None:
        L.check(L.lib().hdg_b200_synchronize(self._ctx))

    def set_jit(self, enabled: bool) -> None:
        """NVRTC-specialised node build for program fields (default on)."""
        L.check(L.lib().hdg_b200_set_jit(self._ctx, int(enabled)))

    def set_rescue_screen(self, screen: float) -> None:
        """Pivot-ratio screen below which an element is re-solved by the reference's
        partial-pivot LU path (kernels_rescue.cuh); >= 1 re-solves every element."""
        L.check(L.lib().hdg_b200_set_rescue_screen(self._ctx, float(screen)))

    def rescued_elements(self) -> int:
        """Elements the last build_condense re-solved by the reference's LU path."""
        n = C.c_int64(0)
        L.check(L.lib().hdg_b200_rescued_elements(self._ctx, C.byref(n)))
        return int(n.value)

    def set_tau_allow_zero(self, enabled: bool) -> None:
        """StabilizationField::allow_zero (element_matrices.hpp:24): accept tau == 0 on
        all faces of an element (negative tau is always rejected, element_matrices.cpp:38-46)."""
        L.check(L.lib().hdg_b200_set_tau_allow_zero(self._ctx, int(enabled)))

    def set_bdm(self, enabled: bool) -> None:
        """BDM variant (bdm_blocks, local_solver.cpp:65-69): u truncated to P_{k-1}, tau ignored."""
        L.check(L.lib().hdg_b200_set_bdm(self._ctx, int(enabled)))

    def set_chat_sparsity(self, enabled: bool) -> bool:
        """K3 skips the structurally zero blocks of Chat_# (default, verified at set_degree);
        False forces the dense kernel. Returns whether the sparse kernel will run."""
        active = C.c_int(0)
        L.check(L.lib().hdg_b200_set_chat_sparsity(self._ctx, int(bool(enabled)), C.byref(active)))
        return bool(active.value)

    def set_recover_variant(self, variant: int) -> None:
        """k = 1..3 recovery kernel: 3 = TMA-streamed cache (default), 2 = direct loads."""
        L.check(L.lib().hdg_b200_set_recover_variant(self._ctx, int(variant)))

    @property
    def jit_status(self) -> str:
        return L.lib().hdg_b200_jit_status(self._ctx).decode()

    def set_timing(self, enabled: bool) -> None:
        L.check(L.lib().hdg_b200_set_timing(self._ctx, int(enabled)))

    def stage_times(self) -> dict:
        """ms per stage since the last query (CUDA events on the engine stream)."""
        ms = (C.c_double * len(L.STAGES))()
        L.check(L.lib().hdg_b200_stage_times(self._ctx, ms))
        return {n: ms[i] for i, n in enumerate(L.STAGES) if ms[i] >= 0}

    # ---------------------------------------------------------------- K1
    def geometry(self, dm: DeviceMesh, tau: Union[float, torch.Tensor] = 1.0,
                 out: Optional[Geometry] = None) -> Geometry:
        n, dev, f64 = dm.nelt, self.device, torch.float64
        g = out or Geometry(torch.empty(n, dtype=f64, device=dev), torch.empty(9, n, dtype=f64, device=dev),
                            torch.empty(12, n, dtype=f64, device=dev),
                            torch.empty(4, n, dtype=torch.int32, device=dev),
                            torch.empty(4, n, dtype=f64, device=dev), torch.empty(12, n, dtype=f64, device=dev),
                            torch.empty(dm.nfc, dtype=f64, device=dev))
        tau_t = tau if isinstance(tau, torch.Tensor) else None
        gs = g.c_struct()
        L.check(L.lib().hdg_b200_geometry(self._ctx, dm.nver, n, dm.nfc, _ptr(dm.coords), _ptr(dm.elements),
                                          _ptr(dm.faces), _ptr(dm.facebyele), _ptr(tau_t),
                                          0.0 if tau_t is not None else float(tau), C.byref(gs)))
        return g

    def upwind_tau(self, g: Geometry, beta: Sequence) -> torch.Tensor:
        tau = torch.empty(4, g.nelt, dtype=torch.float64, device=self.device)
        fs = [as_field(b) for b in beta]
        gs = g.c_struct()
        L.check(L.lib().hdg_b200_upwind_tau(self._ctx, g.nelt, C.byref(gs), fs[0].c_struct(), fs[1].c_struct(),
                                            fs[2].c_struct(), _ptr(tau)))
        return tau

    def quad_points(self, g: Geometry, which: int = 0):
        nq = self.dims["nq" if which == 0 else "nq_post"]
        X, Y, Z = (torch.empty(g.nelt, nq, dtype=torch.float64, device=self.device) for _ in range(3))
        gs = g.c_struct()
        L.check(L.lib().hdg_b200_quad_points(self._ctx, g.nelt, C.byref(gs), which, _ptr(X), _ptr(Y), _ptr(Z)))
        return X, Y, Z

    # ---------------------------------------------------------- K2 + K3
    def alloc_condensed(self, nelt: int, factors: bool = True) -> CondensedSystem:
        d = self.dims
        m = 4 * d["d2"]
        dev, f64 = self.device, torch.float64
        return CondensedSystem(torch.empty(nelt * m * m, dtype=f64, device=dev),
                               torch.empty(nelt * m, dtype=f64, device=dev),
                               torch.empty(nelt * d["factors"], dtype=f64, device=dev) if factors else None, m)

    def work_buffer(self, nelt: int) -> torch.Tensor:
        nbytes = L.lib().hdg_b200_work_size(self._ctx, nelt)
        return torch.empty((nbytes + 7) // 8, dtype=torch.float64, device=self.device)

    def build_condense(self, g: Geometry, kappa, c, f, out: Optional[CondensedSystem] = None,
                       work: Optional[torch.Tensor] = None, check: bool = True) -> CondensedSystem:
        """build_element_matrices -> local_blocks -> condense, fused (local_solver.cpp:71-100)."""
        cs = out or self.alloc_condensed(g.nelt)
        fk, fc, ff = as_field(kappa), as_field(c), as_field(f)
        gs = g.c_struct()
        bad = C.c_int64(-1)
        st = L.lib().hdg_b200_build_condense(self._ctx, g.nelt, C.byref(gs), fk.c_struct(), fc.c_struct(),
                                             ff.c_struct(), _ptr(cs.C), _ptr(cs.Cf), _ptr(cs.factors),
                                             _ptr(work), C.byref(bad) if check else None)
        L.check(st, bad.value)
        return cs

    # ---------------------------------------------------------------- K5
    def recover(self, g: Geometry, dm: DeviceMesh, cs: CondensedSystem, uhat: torch.Tensor,
                out: Optional[LocalSolution] = None) -> LocalSolution:
        """gather_traces + local_recover (global_system.cpp:167-175, local_solver.cpp:102-135)."""
        d3 = self.dims["d3"]
        if out is None:
            out = LocalSolution(*(torch.empty(g.nelt, d3, dtype=torch.float64, device=self.device)
                                  for _ in range(4)))
        gs = g.c_struct()
        L.check(L.lib().hdg_b200_recover(self._ctx, g.nelt, C.byref(gs), _ptr(dm.facebyele), _ptr(cs.factors),
                                         _ptr(uhat), _ptr(out.qx), _ptr(out.qy), _ptr(out.qz), _ptr(out.u)))
        return out

    # ---------------------------------------------------------------- K4
    def pattern(self, mesh: HostMesh, csr: bool = True) -> DevicePattern:
        return self.pattern_from_arrays(*mesh.pattern(), csr=csr)

    def expand(self, coords, elements, dirichlet, neumann) -> DeviceMesh:
        """mesh.cpp:74-171 on the GPU (bit-exact with HostMesh.expand): the raw mesh
        (reference shapes: coords nver x 3, elements nelt x 4, dirichlet/neumann
        rows x 3; numpy or torch) -> DeviceMesh with faces, facetype, facebyele."""
        dev = self.device

        def soa(a, dt):
            t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a))
            return t.to(dev, dt).reshape(-1, t.shape[-1] if t.dim() == 2 else 3).t().contiguous()

        X, E = soa(coords, torch.float64), soa(elements, torch.int32)
        Dr, Nr = soa(dirichlet, torch.int32), soa(neumann, torch.int32)
        nver, nelt, ndir, nneu = X.shape[1], E.shape[1], Dr.shape[1], Nr.shape[1]
        nfc = (4 * nelt + ndir + nneu) // 2
        faces = torch.empty(3, nfc, dtype=torch.int32, device=dev)
        ftype = torch.empty(nfc, dtype=torch.uint8, device=dev)
        fbe = torch.empty(4, nelt, dtype=torch.int32, device=dev)
        out = C.c_int()
        L.check(L.lib().hdg_b200_expand_device(self._ctx, nver, _ptr(X), nelt, _ptr(E), ndir, _ptr(Dr) if ndir else None,
                                               nneu, _ptr(Nr) if nneu else None, _ptr(faces), _ptr(ftype), _ptr(fbe),
                                               C.byref(out)))
        return DeviceMesh(nver, nelt, out.value, X, E, faces, fbe, ftype, ndir, nneu)

    def pattern_device(self, dm: DeviceMesh, csr: bool = True) -> DevicePattern:
        """Skeleton sparsity built on the GPU from dm.facebyele (== HostMesh.pattern())."""
        dev = self.device
        fb = torch.empty(dm.nfc + 1, dtype=torch.int64, device=dev)
        nb = torch.empty(dm.nfc, 8, dtype=torch.int32, device=dev)
        sl = torch.empty(dm.nelt, 16, dtype=torch.uint8, device=dev)
        mx = C.c_int()
        L.check(L.lib().hdg_b200_pattern_device(self._ctx, dm.nelt, dm.nfc, _ptr(dm.facebyele), _ptr(fb), _ptr(nb),
                                                _ptr(sl), C.byref(mx)))
        p = DevicePattern(fb, nb, sl)
        if csr:
            d2 = self.dims["d2"]
            nnz = int(fb[-1].item()) * d2 * d2
            p.rowptr = torch.empty(dm.nfc * d2 + 1, dtype=torch.int64, device=dev)
            p.colidx = torch.empty(nnz, dtype=torch.int32, device=dev)
            L.check(L.lib().hdg_b200_pattern_fill(self._ctx, dm.nfc, d2, _ptr(fb), _ptr(nb), _ptr(p.rowptr),
                                                  _ptr(p.colidx)))
        return p

    def pattern_from_arrays(self, fb: np.ndarray, nb: np.ndarray, sl: np.ndarray, csr: bool = True) -> DevicePattern:
        """Device pattern from (facebase, nbr, slot), e.g. partition.slab_pattern."""
        dev = self.device
        p = DevicePattern(torch.from_numpy(fb).to(dev), torch.from_numpy(nb).to(dev), torch.from_numpy(sl).to(dev))
        if csr:
            d2 = self.dims["d2"]
            nfc = nb.shape[0]
            nnz = int(fb[-1]) * d2 * d2
            p.rowptr = torch.empty(nfc * d2 + 1, dtype=torch.int64, device=dev)
            p.colidx = torch.empty(nnz, dtype=torch.int32, device=dev)
            L.check(L.lib().hdg_b200_pattern_fill(self._ctx, nfc, d2, _ptr(p.facebase), _ptr(p.nbr),
                                                  _ptr(p.rowptr), _ptr(p.colidx)))
        return p

    def face_sides(self, dm: DeviceMesh) -> torch.Tensor:
        """(nfc, 2) int32: e*4+l of each face's elements, lower element first, -1 if one-sided."""
        sides = torch.empty(dm.nfc, 2, dtype=torch.int32, device=self.device)
        L.check(L.lib().hdg_b200_face_sides(self._ctx, dm.nelt, dm.nfc, _ptr(dm.facebyele), _ptr(sides)))
        return sides

    def assemble(self, dm: DeviceMesh, pat: DevicePattern, cs: CondensedSystem,
                 out: Optional[SkeletonSystem] = None, by: str = "faces") -> SkeletonSystem:
        """global_system.cpp:31-56: CSR values of H and b = sum Cf.
        by="faces": each face's block row gathered and written once (no zero fill);
        by="elements": each element's C slice scattered (atomics on the diagonal blocks)."""
        d2 = self.dims["d2"]
        nnz = int(pat.facebase[-1].item()) * d2 * d2 if out is None else out.vals.numel()
        if by == "faces":
            if out is None:
                out = SkeletonSystem(pat.rowptr, pat.colidx,
                                     torch.empty(nnz, dtype=torch.float64, device=self.device),
                                     torch.empty(dm.nfc * d2, dtype=torch.float64, device=self.device), d2)
            if pat.sides is None:
                pat.sides = self.face_sides(dm)
            L.check(L.lib().hdg_b200_scatter_faces(self._ctx, dm.nfc, d2, _ptr(pat.sides), _ptr(pat.slot),
                                                   _ptr(pat.facebase), _ptr(cs.C), _ptr(cs.Cf), _ptr(out.vals),
                                                   _ptr(out.b)))
            return out
        if out is None:
            out = SkeletonSystem(pat.rowptr, pat.colidx, torch.zeros(nnz, dtype=torch.float64, device=self.device),
                                 torch.zeros(dm.nfc * d2, dtype=torch.float64, device=self.device), d2)
        else:
            out.vals.zero_()
            out.b.zero_()
        L.check(L.lib().hdg_b200_scatter(self._ctx, dm.nelt, d2, _ptr(dm.facebyele), _ptr(pat.slot),
                                         _ptr(pat.facebase), _ptr(cs.C), _ptr(cs.Cf), _ptr(out.vals), _ptr(out.b)))
        return out

    # ---------------------------------------------------------------- K9
    def solve_skeleton(self, dm: DeviceMesh, pat: DevicePattern, sys: SkeletonSystem, ub: torch.Tensor,
                       rtol: float = 1e-13, maxit: int = 200000, out: Optional[torch.Tensor] = None):
        """solve_skeleton (global_system.cpp:106-165) on the GPU: Dirichlet dofs = ub, free dofs
        by block-Jacobi CG (symmetric system) or BiCGStab (any other, the reference's SparseLU
        branch) to ||r|| <= rtol ||r0||. Returns (uhat, info)."""
        d2 = sys.d2
        if out is None:
            out = torch.empty(dm.nfc * d2, dtype=torch.float64, device=self.device)
        info = L.hdg_solve_info()
        ubc = ub.contiguous() if dm.ndir else None
        L.check(L.lib().hdg_b200_solve_skeleton(self._ctx, dm.nfc, d2, _ptr(pat.facebase), _ptr(pat.nbr),
                                                _ptr(sys.vals), _ptr(sys.b), dm.ndir, _ptr(ubc), float(rtol),
                                                int(maxit), _ptr(out), C.byref(info)))
        return out, {f: getattr(info, f) for f, _ in info._fields_}

    # ---------------------------------------------------------------- K6
    def postprocess_star(self, g: Geometry, kappa, ls: LocalSolution,
                         out: Optional[torch.Tensor] = None) -> torch.Tensor:
        d31 = self.dims["d3_post"]
        if out is None:
            out = torch.empty(g.nelt, d31, dtype=torch.float64, device=self.device)
        fk = as_field(kappa)
        gs = g.c_struct()
        L.check(L.lib().hdg_b200_postprocess(self._ctx, g.nelt, C.byref(gs), fk.c_struct(), _ptr(ls.qx),
                                             _ptr(ls.qy), _ptr(ls.qz), _ptr(ls.u), _ptr(out)))
        return out

    # ------------------------------------------------- error functionals
    def set_error_rule(self, deg: int = -1) -> None:
        """Tables of degree k and k+1 on tet/tri_rule(deg) (default 2k+4, postprocess.cpp:182-183)."""
        L.check(L.lib().hdg_b200_set_error_rule(self._ctx, int(deg)))

    def hdg_project(self, g: Geometry, q: Sequence, u) -> LocalSolution:
        """hdg_project (postprocess.cpp:95-176): HDG projection of (q, u) into P_k."""
        d3 = self.dims["d3"]
        out = LocalSolution(*(torch.empty(g.nelt, d3, dtype=torch.float64, device=self.device) for _ in range(4)))
        fs = [as_field(x) for x in q] + [as_field(u)]
        gs = g.c_struct()
        bad = C.c_int64(-1)
        st = L.lib().hdg_b200_hdg_project(self._ctx, g.nelt, C.byref(gs), fs[0].c_struct(), fs[1].c_struct(),
                                          fs[2].c_struct(), fs[3].c_struct(), _ptr(out.qx), _ptr(out.qy),
                                          _ptr(out.qz), _ptr(out.u), C.byref(bad))
        L.check(st, bad.value)
        return out

    def compute_errors(self, dm: DeviceMesh, g: Geometry, q: Sequence, u, uhat: torch.Tensor, ls: LocalSolution,
                       ustar: Optional[torch.Tensor] = None) -> dict:
        """compute_errors (postprocess.cpp:178-250) on the GPU: e_q, e_u, e_uhat, eps_u, eps_uhat, e_star."""
        fs = [as_field(x) for x in q] + [as_field(u)]
        gs = g.c_struct()
        rep = L.hdg_error_report()
        L.check(L.lib().hdg_b200_compute_errors(self._ctx, g.nelt, C.byref(gs), dm.nver, _ptr(dm.coords), dm.nfc,
                                                _ptr(dm.faces), fs[0].c_struct(), fs[1].c_struct(),
                                                fs[2].c_struct(), fs[3].c_struct(), _ptr(uhat), _ptr(ls.qx),
                                                _ptr(ls.qy), _ptr(ls.qz), _ptr(ls.u), _ptr(ustar), C.byref(rep)))
        return {f: getattr(rep, f) for f, _ in rep._fields_}

    # ---------------------------------------------------------------- K8
    def dirichlet_project(self, dm: DeviceMesh, g, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """dirichlet_project (global_system.cpp:58-70): (ndir, d2), row j = Dirichlet face j."""
        d2 = self.dims["d2"]
        if out is None:
            out = torch.empty(dm.ndir, d2, dtype=torch.float64, device=self.device)
        fg = as_field(g)
        L.check(L.lib().hdg_b200_dirichlet_project(self._ctx, dm.nver, _ptr(dm.coords), dm.nfc, _ptr(dm.faces),
                                                   dm.ndir, fg.c_struct(), _ptr(out)))
        return out

    def skeleton_project(self, dm: DeviceMesh, g, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """l2_project_skeleton (postprocess.cpp:84-93): (nfc, d2), dof f*d2 + i."""
        d2 = self.dims["d2"]
        if out is None:
            out = torch.empty(dm.nfc, d2, dtype=torch.float64, device=self.device)
        fg = as_field(g)
        L.check(L.lib().hdg_b200_skeleton_project(self._ctx, dm.nver, _ptr(dm.coords), dm.nfc, _ptr(dm.faces),
                                                  fg.c_struct(), _ptr(out)))
        return out

    def neumann_load(self, dm: DeviceMesh, g: Geometry, q: Sequence, b: Optional[torch.Tensor] = None,
                     alpha: float = 1.0) -> torch.Tensor:
        """neumann_load (global_system.cpp:72-104) of the vector field q = (qx, qy, qz):
        b[f*d2 + i] += alpha * <q . n, D_i>_f on the Neumann faces. With b None a zeroed
        vector is returned (the reference's value); alpha=-1 on the assembled b is
        study.cpp:25."""
        d2 = self.dims["d2"]
        if b is None:
            b = torch.zeros(dm.nfc * d2, dtype=torch.float64, device=self.device)
        fs = [as_field(x) for x in q]
        gs = g.c_struct()
        L.check(L.lib().hdg_b200_neumann_load(self._ctx, dm.nver, _ptr(dm.coords), dm.nfc, _ptr(dm.faces),
                                              dm.nelt, _ptr(dm.facebyele), C.byref(gs), dm.ndir, dm.nneu,
                                              fs[0].c_struct(), fs[1].c_struct(), fs[2].c_struct(),
                                              float(alpha), _ptr(b)))
        return b

    # ---------------------------------------------------------------- K7
    def convection_bilinear_matrices(self, g: Geometry, beta: Sequence, out=None):
        """convection_bilinear_matrices (convdiff.cpp:5-28): (vol, dp, dd) Batch3 views;
        out = (vol, dp, dd) flat buffers from a previous call's .base tensors to reuse."""
        d = self.dims
        d3, m, n = d["d3"], 4 * d["d2"], g.nelt
        if out is None:
            vol = torch.empty(n * d3 * d3, dtype=torch.float64, device=self.device)
            dp = torch.empty(n * m * d3, dtype=torch.float64, device=self.device)
            dd = torch.empty(n * m * m, dtype=torch.float64, device=self.device)
        else:
            vol, dp, dd = out
        fs = [as_field(b) for b in beta]
        gs = g.c_struct()
        L.check(L.lib().hdg_b200_convection_block(self._ctx, n, C.byref(gs), fs[0].c_struct(), fs[1].c_struct(),
                                                  fs[2].c_struct(), _ptr(vol), _ptr(dp), _ptr(dd)))
        return (vol.view(n, d3, d3).transpose(1, 2), dp.view(n, d3, m).transpose(1, 2),
                dd.view(n, m, m).transpose(1, 2))

    def element_matrices(self, g: Geometry, kappa, c, f):
        """The ElementMatrixSet of build_element_matrices, materialised (parity/debug)."""
        d = self.dims
        d3, m, n = d["d3"], 4 * d["d2"], g.nelt
        shapes = dict(Mkinv=(d3, d3), Mc=(d3, d3), Cx=(d3, d3), Cy=(d3, d3), Cz=(d3, d3), tauPP=(d3, d3),
                      tauDP=(m, d3), nxDP=(m, d3), nyDP=(m, d3), nzDP=(m, d3), tauDD=(m, m), fvec=(d3, 1))
        bufs = {k: torch.empty(n * r * cc, dtype=torch.float64, device=self.device) for k, (r, cc) in shapes.items()}
        em = L.hdg_element_matrices()
        for k, t in bufs.items():
            setattr(em, k, t.data_ptr())
        fk, fc, ff = as_field(kappa), as_field(c), as_field(f)
        gs = g.c_struct()
        L.check(L.lib().hdg_b200_element_matrices(self._ctx, n, C.byref(gs), fk.c_struct(), fc.c_struct(),
                                                  ff.c_struct(), C.byref(em)))
        out = {k: bufs[k].view(n, cc, r).transpose(1, 2) for k, (r, cc) in shapes.items() if k != "fvec"}
        out["fvec"] = bufs["fvec"].view(n, d3)
        return out
