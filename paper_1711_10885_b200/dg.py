"""Thin Python binding of libdg_b200.so (include/dg.h): argument marshalling only.

Every step of y = A z runs in the library's CUDA kernels; there is no CPU or
PyTorch fallback. If the shared library is missing this module raises at import
of the library handle (DGError), loudly.

Device vectors are torch CUDA float64 tensors (torch provides memory, streams and
process groups only); host vectors for apply_host are numpy float64 arrays.
"""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DG_LIB") or os.path.join(HERE, "libdg_b200.so")

DG_OK, DG_EINVAL, DG_ENOMEM, DG_ECUDA, DG_ENCCL, DG_EUNSUPPORTED = 0, -1, -2, -3, -4, -5
VOLUME, INTERIOR_FACES, BOUNDARY_FACES, ALL, HALO_EXTERNAL = 1, 2, 4, 7, 0x100
BC_DIRICHLET, BC_PERIODIC = 0, 1

EXPORTED = ["dg_setup", "dg_local_layout", "dg_apply", "dg_apply_ex", "dg_residual", "dg_apply_host",
            "dg_sync", "dg_destroy", "dg_strerror", "dg_halo_info", "dg_halo_buffer", "dg_halo_pack",
            "dg_fill_uniform", "dg_fill_uniform_local", "dg_nccl_unique_id", "dg_get_kernel_info", "dg_partition",
            "dg_set_diffusion", "dg_fill_uniform_cells", "dg_ssp_stage", "dg_set_velocity", "dg_set_quadrature",
            "dg_set_affine", "dg_matrix_size", "dg_assemble", "dg_matrix_apply", "dg_fabric_id", "dg_comm_info",
            "dg_set_geometry", "dg_fabric_id_direct", "dg_p2p_blob_bytes", "dg_p2p_export", "dg_p2p_import",
            "dg_timeline"]


class DGError(RuntimeError):
    def __init__(self, code, what=""):
        self.code = code
        msg = _lib.dg_strerror(code).decode() if _lib is not None else str(code)
        super().__init__("%s: %s (%d)" % (what, msg, code))


class MeshDesc(ctypes.Structure):
    _fields_ = [("ncells", ctypes.c_int64 * 3), ("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3),
                ("bc", ctypes.c_int * 6), ("parts", ctypes.c_int * 3)]


class KernelInfo(ctypes.Structure):
    _fields_ = [("launches_per_apply", ctypes.c_int), ("cells_per_cta", ctypes.c_int),
                ("threads_per_cta", ctypes.c_int), ("smem_bytes", ctypes.c_int),
                ("regs_per_thread", ctypes.c_int), ("ctas_per_sm", ctypes.c_int)]


_lib = None


def lib():
    """The loaded library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError("libdg_b200.so not built: run `python -m paper_1711_10885_b200.build` "
                               "(there is no fallback path)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64
        L.dg_setup.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(MeshDesc), ctypes.c_int, vp, vp, ctypes.c_double,
                               ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp]
        L.dg_local_layout.argtypes = [vp, vp, vp, vp]
        L.dg_apply.argtypes = [vp, vp, vp, vp]
        L.dg_apply_ex.argtypes = [vp, vp, vp, ctypes.c_uint, vp]
        L.dg_residual.argtypes = [vp, vp, vp, vp, vp]
        L.dg_apply_host.argtypes = [vp, vp, vp]
        L.dg_sync.argtypes = [vp]
        L.dg_destroy.argtypes = [vp]
        L.dg_strerror.argtypes = [ctypes.c_int]
        L.dg_strerror.restype = ctypes.c_char_p
        L.dg_halo_info.argtypes = [vp, ctypes.c_int, vp, vp]
        L.dg_halo_buffer.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp]
        L.dg_halo_pack.argtypes = [vp, vp, vp]
        L.dg_fill_uniform.argtypes = [vp, i64, u64, i64, vp]
        L.dg_fill_uniform_local.argtypes = [vp, vp, u64, vp]
        L.dg_nccl_unique_id.argtypes = [vp]
        L.dg_fabric_id.argtypes = [vp]
        L.dg_comm_info.argtypes = [vp, vp, vp]
        L.dg_timeline.argtypes = [vp, ctypes.c_int, vp, ctypes.c_int]
        L.dg_set_geometry.argtypes = [vp, vp, ctypes.c_int, vp]
        L.dg_fabric_id_direct.argtypes = [vp]
        L.dg_p2p_blob_bytes.argtypes = []
        L.dg_p2p_export.argtypes = [vp, vp]
        L.dg_p2p_import.argtypes = [vp, vp, ctypes.c_char_p]
        L.dg_get_kernel_info.argtypes = [vp, ctypes.POINTER(KernelInfo)]
        L.dg_partition.argtypes = [ctypes.POINTER(MeshDesc), ctypes.c_int, ctypes.c_int, vp, vp, vp]
        L.dg_set_diffusion.argtypes = [vp, vp, ctypes.c_uint, vp]
        L.dg_fill_uniform_cells.argtypes = [vp, vp, ctypes.c_int, u64, vp]
        L.dg_set_velocity.argtypes = [vp, ctypes.c_int, vp]
        L.dg_set_affine.argtypes = [vp, vp]
        L.dg_set_quadrature.argtypes = [vp, ctypes.c_int]
        L.dg_matrix_size.argtypes = [vp, vp]
        L.dg_assemble.argtypes = [vp, vp, vp]
        L.dg_matrix_apply.argtypes = [vp, vp, vp, vp, vp]
        L.dg_ssp_stage.argtypes = [vp, vp, vp, vp, ctypes.c_double, ctypes.c_double, ctypes.c_double, vp, vp]
        for name in EXPORTED:
            if name != "dg_strerror":
                getattr(L, name).restype = ctypes.c_int
        L.dg_p2p_blob_bytes.restype = ctypes.c_size_t
        _lib = L
    return _lib


def _check(rc, what):
    if rc != DG_OK:
        raise DGError(rc, what)


def _ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dev_vec(t, n, name):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise TypeError("%s must be a contiguous CUDA float64 tensor" % name)
    if t.numel() != n:
        raise ValueError("%s has %d entries, expected %d" % (name, t.numel(), n))
    if t.data_ptr() % 16:
        raise ValueError("%s must be 16-byte aligned (the kernels use 16-byte vector accesses)" % name)


def nccl_unique_id():
    buf = (ctypes.c_ubyte * 128)()
    _check(lib().dg_nccl_unique_id(buf), "dg_nccl_unique_id")
    return bytes(buf)


def fabric_id():
    """Id of an in-process fabric group (dg_fabric_id): the ranks of a partitioned operator as
    threads of this process, e.g. P ranks on one GPU for a test of the partitioned path."""
    buf = (ctypes.c_ubyte * 128)()
    _check(lib().dg_fabric_id(buf), "dg_fabric_id")
    return bytes(buf)


def fabric_id_direct():
    """Id of an in-process fabric group whose applies use the direct (fused) halo: each rank's trace
    pack stores into the neighbours' receive buffers (dg_fabric_id_direct)."""
    buf = (ctypes.c_ubyte * 128)()
    _check(lib().dg_fabric_id_direct(buf), "dg_fabric_id_direct")
    return bytes(buf)


def p2p_attach(op, shm_name=None, group=None):
    """Switch a partitioned NCCL operator (one process per GPU) to the direct (fused) halo over CUDA
    IPC: export this rank's blob, all-gather the blobs through torch.distributed, import them
    (dg_p2p_export / dg_p2p_import). Collective."""
    import os as _os
    import torch.distributed as dist
    n = lib().dg_p2p_blob_bytes()
    blob = (ctypes.c_ubyte * n)()
    _check(lib().dg_p2p_export(op._h, blob), "dg_p2p_export")
    world = dist.get_world_size(group)
    if shm_name is None:
        name = ["/dg_p2p_%d_%d" % (_os.getpid(), id(op))] if dist.get_rank(group) == 0 else [None]
        dist.broadcast_object_list(name, src=0, group=group)
        shm_name = name[0]
    blobs = [None] * world
    dist.all_gather_object(blobs, bytes(blob), group=group)
    allb = (ctypes.c_ubyte * (n * world)).from_buffer_copy(b"".join(blobs))
    _check(lib().dg_p2p_import(op._h, allb, shm_name.encode()), "dg_p2p_import")
    return shm_name


def mesh_desc(ncells, lo, hi, parts=(1, 1, 1), bc=(BC_DIRICHLET,) * 6):
    m = MeshDesc()
    for q in range(3):
        m.ncells[q] = int(ncells[q])
        m.lo[q] = float(lo[q])
        m.hi[q] = float(hi[q])
        m.parts[q] = int(parts[q])
    for f in range(6):
        m.bc[f] = int(bc[f])
    return m


def bc_from_periodic(periodic):
    """bc[6] with both sides of every periodic direction glued, the others Dirichlet."""
    return tuple(BC_PERIODIC if periodic[f >> 1] else BC_DIRICHLET for f in range(6))


def partition(ncells, parts, rank, periodic=(0, 0, 0)):
    """Host-only block partition (dg_partition): (cell_lo, cell_cnt, neighbour rank per face)."""
    m = mesh_desc(ncells, (0, 0, 0), (1, 1, 1), parts, bc_from_periodic(periodic))
    lo = (ctypes.c_int64 * 3)()
    cnt = (ctypes.c_int64 * 3)()
    nb = (ctypes.c_int * 6)()
    nr = int(parts[0]) * int(parts[1]) * int(parts[2])
    _check(lib().dg_partition(ctypes.byref(m), int(rank), nr, lo, cnt, nb), "dg_partition")
    return tuple(lo), tuple(cnt), tuple(nb)


def fill_uniform(t, seed, offset=0, stream=None):
    """t[i] = U(seed, offset + i) on the device (reading C-13)."""
    _check(lib().dg_fill_uniform(_ptr(t), t.numel(), seed, offset, _stream(stream)), "dg_fill_uniform")


class Operator:
    """One dg_ctx: the SIPG operator on this rank's block of a structured box mesh."""

    def __init__(self, ncells, lo, hi, k, D, b, c, sigma, device=0, rank=0, nranks=1, parts=(1, 1, 1),
                 nccl_id=None, bc=(BC_DIRICHLET,) * 6):
        L = lib()
        m = mesh_desc(ncells, lo, hi, parts, bc)
        Dm = (ctypes.c_double * 9)(*[float(v) for v in np.asarray(D, dtype=np.float64).ravel()])
        bv = (ctypes.c_double * 3)(*[float(v) for v in b])
        idbuf = None
        if nccl_id is not None:
            idbuf = (ctypes.c_ubyte * 128).from_buffer_copy(bytes(nccl_id))
        h = ctypes.c_void_p()
        _check(L.dg_setup(ctypes.byref(h), ctypes.byref(m), int(k), Dm, bv, float(c), float(sigma), int(device),
                          int(rank), int(nranks), idbuf), "dg_setup")
        self._h = h
        self.k = k
        self.n3 = (k + 1) ** 3
        self.device = device
        lo_ = (ctypes.c_int64 * 3)()
        cnt = (ctypes.c_int64 * 3)()
        nd = ctypes.c_int64()
        _check(L.dg_local_layout(h, lo_, cnt, ctypes.byref(nd)), "dg_local_layout")
        self.cell_lo = tuple(lo_)
        self.cell_cnt = tuple(cnt)
        self.ndofs = nd.value

    # -- compute ------------------------------------------------------------------------------------
    def apply(self, z, y, terms=ALL, stream=None):
        """y = A z (dg_apply), or the parts of A in `terms` (dg_apply_ex)."""
        _dev_vec(z, self.ndofs, "z")
        _dev_vec(y, self.ndofs, "y")
        if terms == ALL:
            _check(lib().dg_apply(self._h, _ptr(z), _ptr(y), _stream(stream)), "dg_apply")
        else:
            _check(lib().dg_apply_ex(self._h, _ptr(z), _ptr(y), terms, _stream(stream)), "dg_apply_ex")
        return y

    def residual(self, z, f, r, stream=None):
        for t, nm in ((z, "z"), (f, "f"), (r, "r")):
            _dev_vec(t, self.ndofs, nm)
        _check(lib().dg_residual(self._h, _ptr(z), _ptr(f), _ptr(r), _stream(stream)), "dg_residual")
        return r

    def ssp_stage(self, z, out, dt, f=None, w=None, a=0.0, b=1.0, stream=None):
        """out = a w + b (z + dt M^-1 (f - A z)) (dg_ssp_stage; M = Delta_T I)."""
        for t, nm in ((z, "z"), (out, "out"), (f, "f"), (w, "w")):
            if t is not None:
                _dev_vec(t, self.ndofs, nm)
        _check(lib().dg_ssp_stage(self._h, _ptr(z), _ptr(f), _ptr(w), float(a), float(b), float(dt), _ptr(out),
                                  _stream(stream)), "dg_ssp_stage")
        return out

    def heun_step(self, u, dt, tmp, out, f=None, stream=None):
        """One SSP-RK2 (Heun, Shu-Osher form) step u -> out; tmp holds the first stage."""
        self.ssp_stage(u, tmp, dt, f=f, stream=stream)
        self.ssp_stage(tmp, out, dt, f=f, w=u, a=0.5, b=0.5, stream=stream)
        return out

    def apply_host(self, z_host, y_host):
        """End-to-end: host arrays in, host array out (copies inside the call)."""
        for a in (z_host, y_host):
            if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous
                    and a.size == self.ndofs):
                raise TypeError("host vectors must be contiguous float64 numpy arrays of ndofs entries")
        _check(lib().dg_apply_host(self._h, a_ptr(z_host), a_ptr(y_host)), "dg_apply_host")
        return y_host

    def matrix_size(self):
        """dg_matrix_size: doubles of the assembled block-stencil matrix (7 n^6 per cell)."""
        n = ctypes.c_int64()
        _check(lib().dg_matrix_size(self._h, ctypes.byref(n)), "dg_matrix_size")
        return n.value

    def assemble(self, A, stream=None):
        """dg_assemble: the operator of the next apply into the caller's device matrix A."""
        _dev_vec(A, self.matrix_size(), "A")
        _check(lib().dg_assemble(self._h, _ptr(A), _stream(stream)), "dg_assemble")

    def matrix_apply(self, A, z, y, stream=None):
        """dg_matrix_apply: y = A z with the assembled matrix."""
        _dev_vec(A, self.matrix_size(), "A")
        _dev_vec(z, self.ndofs, "z")
        _dev_vec(y, self.ndofs, "y")
        _check(lib().dg_matrix_apply(self._h, _ptr(A), _ptr(z), _ptr(y), _stream(stream)), "dg_matrix_apply")
        return y

    def set_diffusion(self, Dcell, flags=0, stream=None):
        """Per-cell tensors: CUDA float64 tensor of local cells x 9 (row-major), or None to
        revert to the constant D of the constructor (dg_set_diffusion)."""
        if Dcell is not None:
            ncell = self.ndofs // self.n3
            _dev_vec(Dcell, ncell * 9, "Dcell")
        _check(lib().dg_set_diffusion(self._h, _ptr(Dcell), flags, _stream(stream)), "dg_set_diffusion")

    def set_affine(self, J):
        """Physical mesh x = lo + J (xhat - lo) of the axis-aligned box (dg_set_affine; NEXT-3)."""
        a = (ctypes.c_double * 9)(*[float(v) for v in np.asarray(J, dtype=np.float64).ravel()])
        _check(lib().dg_set_affine(self._h, a), "dg_set_affine")

    def set_geometry(self, vert, m=None, stream=None):
        """Multilinear mesh (dg_set_geometry; NEXT-3): vert = the padded vertex grid of this rank's
        box, (nloc+3)^3 x 3 doubles (CUDA float64 tensor or numpy array), or None to revert;
        m Gauss points per direction (default k+1)."""
        if vert is None:
            _check(lib().dg_set_geometry(self._h, None, 0, _stream(stream)), "dg_set_geometry")
            return
        cnt = (self.cell_cnt[0] + 3) * (self.cell_cnt[1] + 3) * (self.cell_cnt[2] + 3) * 3
        if isinstance(vert, np.ndarray):
            vert = np.ascontiguousarray(vert, dtype=np.float64)
            if vert.size != cnt:
                raise ValueError("vert has %d entries, expected %d" % (vert.size, cnt))
            ptr = a_ptr(vert)
        else:
            _dev_vec(vert, cnt, "vert")
            ptr = _ptr(vert)
        _check(lib().dg_set_geometry(self._h, ptr, int(m if m else self.k + 1), _stream(stream)),
               "dg_set_geometry")

    def set_velocity(self, kind, amp=(1.0, 1.0, 1.0)):
        """Velocity field b(x) at every quadrature point: 0 constant, 1 Taylor-Green, 2 linear (dg_set_velocity)."""
        a = (ctypes.c_double * 3)(*[float(v) for v in amp])
        _check(lib().dg_set_velocity(self._h, int(kind), a), "dg_set_velocity")

    def set_quadrature(self, m):
        """Gauss points per direction (k+1 or k+3; dg_set_quadrature)."""
        _check(lib().dg_set_quadrature(self._h, int(m)), "dg_set_quadrature")

    def fill_uniform_cells(self, t, per_cell, seed, stream=None):
        """t[per_cell * l + i] = U(seed, per_cell * e_global(l) + i) (dg_fill_uniform_cells)."""
        _dev_vec(t, self.ndofs // self.n3 * per_cell, "t")
        _check(lib().dg_fill_uniform_cells(self._h, _ptr(t), per_cell, seed, _stream(stream)),
               "dg_fill_uniform_cells")

    def set_tensor_field(self, seed, stream=None):
        """The seeded Problem A tensor field (inputs.tensor_field_from_uniforms) of this rank's cells."""
        import torch
        from . import inputs
        ncell = self.ndofs // self.n3
        u6 = torch.empty(ncell * 6, dtype=torch.float64, device="cuda:%d" % self.device)
        self.fill_uniform_cells(u6, 6, seed, stream)
        D9 = inputs.tensor_field_from_uniforms(u6.view(ncell, 6))
        self.set_diffusion(D9.view(-1), stream=stream)
        del u6, D9

    def fill_uniform_local(self, t, seed, stream=None):
        _dev_vec(t, self.ndofs, "t")
        _check(lib().dg_fill_uniform_local(self._h, _ptr(t), seed, _stream(stream)), "dg_fill_uniform_local")

    # -- halo ---------------------------------------------------------------------------------------
    def halo_info(self, face):
        r = ctypes.c_int()
        c = ctypes.c_int64()
        _check(lib().dg_halo_info(self._h, face, ctypes.byref(r), ctypes.byref(c)), "dg_halo_info")
        return r.value, c.value

    def halo_buffer_ptr(self, face, which):
        p = ctypes.c_void_p()
        _check(lib().dg_halo_buffer(self._h, face, which, ctypes.byref(p)), "dg_halo_buffer")
        return p.value

    def halo_pack(self, z, stream=None):
        _check(lib().dg_halo_pack(self._h, _ptr(z), _stream(stream)), "dg_halo_pack")

    def comm_info(self):
        """(transport, nranks): transport 'none' | 'nccl' | 'fabric' | 'fabric-direct' | 'p2p-ipc', nranks as
        the communicator reports."""
        t, n = ctypes.c_int(), ctypes.c_int()
        _check(lib().dg_comm_info(self._h, ctypes.byref(t), ctypes.byref(n)), "dg_comm_info")
        return ("none", "nccl", "fabric", "fabric-direct", "p2p-ipc")[t.value], n.value

    def timeline_arm(self):
        """Record timing events around the launches of the next (partitioned) apply (dg_timeline)."""
        _check(lib().dg_timeline(self._h, 1, None, 0), "dg_timeline")

    def timeline(self):
        """ms since the armed apply's start: pack (+ exchange) begin / end on the comm stream, inner
        kernel begin / end, shell kernel start / end (waits for that apply)."""
        t = (ctypes.c_double * 6)()
        _check(lib().dg_timeline(self._h, 0, t, 6), "dg_timeline")
        keys = ("pack_begin", "pack_end", "inner_begin", "inner_end", "shell_begin", "shell_end")
        return dict(zip(keys, list(t)))

    # -- info / lifetime ----------------------------------------------------------------------------
    def kernel_info(self):
        ki = KernelInfo()
        _check(lib().dg_get_kernel_info(self._h, ctypes.byref(ki)), "dg_get_kernel_info")
        return {f: getattr(ki, f) for f, _ in KernelInfo._fields_}

    def sync(self):
        _check(lib().dg_sync(self._h), "dg_sync")

    def close(self):
        if getattr(self, "_h", None):
            rc = lib().dg_destroy(self._h)
            self._h = None
            _check(rc, "dg_destroy")

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def a_ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


def from_config(cfg, **kw):
    """Operator for a configs.Config: boundary conditions, velocity field and quadrature applied
    (a per-cell tensor field is left to set_tensor_field)."""
    if getattr(cfg, "periodic", (0, 0, 0)) != (0, 0, 0) and "bc" not in kw:
        kw["bc"] = bc_from_periodic(cfg.periodic)
    op = Operator(cfg.ncells, cfg.lo, cfg.hi, cfg.k, cfg.D, cfg.b, cfg.c, cfg.sigma, **kw)
    if getattr(cfg, "bkind", 0):
        op.set_velocity(cfg.bkind)
    if getattr(cfg, "geo_amp", 0.0) > 0.0:
        op.set_geometry(padded_vertex_grid(cfg, op.cell_lo, op.cell_cnt), cfg.m or cfg.k + 1)
    elif getattr(cfg, "m", 0) and cfg.m != cfg.k + 1:
        op.set_quadrature(cfg.m)
    return op


def padded_vertex_grid(cfg, cell_lo, cell_cnt):
    """The padded vertex grid dg_set_geometry takes for a rank's box (include/dg.h), from the
    seeded multilinear mesh of a config (inputs.vertex_grid)."""
    from . import inputs
    box = (tuple(cell_lo[q] - 1 for q in range(3)), tuple(cell_lo[q] + cell_cnt[q] + 2 for q in range(3)))
    return inputs.vertex_grid(cfg.ncells, cfg.lo, cfg.hi, cfg.geo_amp, cfg.geo_seed, cfg.periodic, box=box)
