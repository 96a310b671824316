"""Multi-GPU: batch sharding and the sharded four-step transform.

Two strategies:

1. Batch sharding (configs 1-4): independent transforms; rank r takes the
   contiguous row block ``shard_rows(batch, world, r)``; no communication.

2. One very long transform over G GPUs (config 5): the sharded four-step
   of the C ABI (``sfft_dist_*``).  With N = N1*N2 (N1 = 2^floor(m/2)):

   * input  x[n], n = N2*n1 + n2, lives on rank n2 // (N2/G) as a local
     [N1, N2/G] array (``scatter_input``);
   * phase 0 (local): stages 1..log2 N1 -- the length-N1 transforms of the
     local columns -- written straight into the all-to-all send layout
     [G, N2/G, N1/G] (one contiguous segment per destination);
   * exchange: one all-to-all per plane (NCCL over NVLink/NVSwitch through
     ``torch.distributed.all_to_all_single``) -- the only collective;
   * phase 1 (local): stages log2 N1 + 1 .. m on the received [N2, N1/G]
     array; output X[k], k = k1 + N1*k2, on rank k1 // (N1/G) as a local
     [N2, N1/G] array (``gather_output``).

   The arithmetic is the reference's radix-2 stages, so an fp64 sharded
   transform is bit-identical to the single-GPU one and to the reference.

   Fused variant (``P2PExchange``): the receive planes live in torch
   symmetric memory and phase 0's last launch stores each destination
   segment straight into that rank's receive planes over NVLink/NVSwitch
   (``DistPlan.phase0_p2p``), so the exchange overlaps the compute tile by
   tile and the send buffer's HBM round trip disappears; two symmetric-memory
   barriers order it.

``fft_dist`` takes an optional ``phase_fn`` so the orchestration (layouts,
exchange, gather) is testable on CPU with gloo (tests/test_dist_gloo.py).
"""

import ctypes
import datetime
import os

import numpy as np
import torch

from . import _ffi
from .transform import _DTYPE_CODE, _resolve_device, _stream_ptr


DEFAULT_TIMEOUT_S = 300


def init_process_group(backend: str = "nccl", device=None, timeout_s: float = DEFAULT_TIMEOUT_S):
    """torch.distributed setup with the failure handling this library relies
    on: a bounded collective timeout (a hung peer raises instead of blocking
    forever), NCCL asynchronous error handling (a failed communicator aborts
    the process rather than leaving it spinning), and NCCL INIT logs on
    stderr so a launcher can confirm the communicator size."""
    import torch.distributed as dist
    os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
    if backend == "nccl":
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    kw = {"timeout": datetime.timedelta(seconds=timeout_s)}
    if backend == "nccl" and device is not None:
        kw["device_id"] = torch.device(device)
    dist.init_process_group(backend, **kw)


def shard_rows(batch: int, world: int, rank: int):
    """[start, end) of rank's contiguous block of rows (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} out of range for world size {world}")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def four_step_split(m: int):
    """(log2 N1, log2 N2) of the sharded schedule."""
    l1 = m // 2
    return l1, m - l1


class DistPlan:
    """Sharded four-step plan for rank ``rank`` of ``world`` (C: sfft_dist_plan)."""

    def __init__(self, m, world, rank, dtype=torch.float32, device=None):
        if dtype not in _DTYPE_CODE:
            raise ValueError(f"dtype must be torch.float32 or torch.float64, got {dtype}")
        self.device = _resolve_device(device)
        self.m, self.world, self.rank, self.dtype = m, world, rank, dtype
        h = ctypes.c_void_p()
        _ffi.check(_ffi.lib.sfft_dist_plan_create(m, _DTYPE_CODE[dtype], world, rank, self.device.index,
                                                  ctypes.byref(h)))
        self._handle = h.value
        local, l1, seg = ctypes.c_int64(), ctypes.c_int(), ctypes.c_int64()
        _ffi.check(_ffi.lib.sfft_dist_layout(self._handle, ctypes.byref(local), ctypes.byref(l1),
                                             ctypes.byref(seg)))
        self.local_elems, self.l1, self.segment_elems = local.value, l1.value, seg.value
        ws = ctypes.c_size_t()
        _ffi.check(_ffi.lib.sfft_dist_workspace_bytes(self._handle, ctypes.byref(ws)))
        self.workspace_bytes = ws.value
        l0, l1_ = ctypes.c_int(), ctypes.c_int()
        _ffi.check(_ffi.lib.sfft_dist_schedule(self._handle, ctypes.byref(l0), ctypes.byref(l1_)))
        # pass-kernel launches of phase 0 / phase 1; each reads and writes the
        # rank's N/G elements of both planes once (the HBM sweeps of a step)
        self.launches = (l0.value, l1_.value)

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h:
            try:
                _ffi.lib.sfft_dist_plan_destroy(h)
            except Exception:
                pass

    @property
    def n1(self):
        return 1 << self.l1

    @property
    def n2(self):
        return 1 << (self.m - self.l1)

    def phase(self, phase, x_re, x_im, y_re, y_im, inverse=False, workspace=None):
        """Run phase 0 (x = local input -> y = send buffer) or phase 1
        (x = receive buffer -> y = local output) on the current stream."""
        for t in (x_re, x_im, y_re, y_im):
            if t.device != self.device or t.dtype != self.dtype or not t.is_contiguous() \
                    or t.numel() != self.local_elems:
                raise ValueError("phase buffers must be contiguous, on the plan's device and dtype, "
                                 f"with {self.local_elems} elements")
        if workspace is None:
            workspace = torch.empty(self.workspace_bytes, dtype=torch.uint8, device=self.device)
        _ffi.check(_ffi.lib.sfft_dist_exec_phase(
            self._handle, phase, x_re.data_ptr(), x_im.data_ptr(), y_re.data_ptr(), y_im.data_ptr(),
            _ffi.SFFT_INVERSE if inverse else _ffi.SFFT_FORWARD, workspace.data_ptr(),
            _stream_ptr(self.device)))
        return y_re, y_im

    def phase0_p2p(self, x_re, x_im, recv_re, recv_im, inverse=False, workspace=None):
        """Phase 0 with the exchange fused in: the last launch stores each
        destination segment straight into rank h's receive planes
        (``recv_re[h]``, ``recv_im[h]``: device tensors or raw device
        pointers of every rank, e.g. symmetric-memory peer buffers)."""
        if len(recv_re) != self.world or len(recv_im) != self.world:
            raise ValueError(f"need {self.world} receive buffers per plane")
        for t in (x_re, x_im):
            if t.device != self.device or t.dtype != self.dtype or not t.is_contiguous() \
                    or t.numel() != self.local_elems:
                raise ValueError("input planes must be contiguous, on the plan's device and dtype, "
                                 f"with {self.local_elems} elements")
        ptr = lambda v: v if isinstance(v, int) else v.data_ptr()   # noqa: E731
        pr = (ctypes.c_void_p * self.world)(*[ptr(v) for v in recv_re])
        pi = (ctypes.c_void_p * self.world)(*[ptr(v) for v in recv_im])
        if workspace is None:
            workspace = torch.empty(self.workspace_bytes, dtype=torch.uint8, device=self.device)
        _ffi.check(_ffi.lib.sfft_dist_exec_phase0_p2p(
            self._handle, x_re.data_ptr(), x_im.data_ptr(), pr, pi, self.world,
            _ffi.SFFT_INVERSE if inverse else _ffi.SFFT_FORWARD, workspace.data_ptr(),
            _stream_ptr(self.device)))


class P2PExchange:
    """Receive planes in torch symmetric memory, so phase 0 can store into
    every peer's buffer directly over NVLink/NVSwitch (the fused exchange).
    One per (plan, process group); ``run`` = barrier, fused phase 0,
    barrier, phase 1."""

    def __init__(self, plan: DistPlan, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        self.plan = plan
        n = plan.local_elems
        self.buf = symm_mem.empty(2 * n, dtype=plan.dtype, device=plan.device)
        grp = group if group is not None else dist.group.WORLD
        self.handle = symm_mem.rendezvous(self.buf, grp)
        esz = self.buf.element_size()
        self.peer_re = [int(p) for p in self.handle.buffer_ptrs]
        self.peer_im = [int(p) + n * esz for p in self.handle.buffer_ptrs]
        self.recv_re, self.recv_im = self.buf[:n], self.buf[n:]

    def run(self, x_re, x_im, y_re, y_im, inverse=False, workspace=None):
        self.handle.barrier(channel=0)          # every rank done reading its receive planes
        with _ffi.nvtx_range("sfft_dist_phase0_p2p"):
            self.plan.phase0_p2p(x_re, x_im, self.peer_re, self.peer_im, inverse=inverse, workspace=workspace)
        self.handle.barrier(channel=0)          # every store landed
        with _ffi.nvtx_range("sfft_dist_phase1"):
            return self.plan.phase(1, self.recv_re, self.recv_im, y_re, y_im, inverse=inverse,
                                   workspace=workspace)


def scatter_input(x, world, rank, l1):
    """Rank's local input block [N1, N2/G] of a global length-N vector x
    (numpy or torch, 1-D): columns n2 of the [N1, N2] view."""
    n = x.shape[0]
    n1 = 1 << l1
    n2 = n // n1
    w = n2 // world
    return x.reshape(n1, n2)[:, rank * w:(rank + 1) * w]


def gather_output(locals_, l1):
    """Global X (length N) from the ranks' local outputs [N2, N1/G]."""
    world = len(locals_)
    lib = np if isinstance(locals_[0], np.ndarray) else torch
    blocks = lib.concatenate(list(locals_), 1) if lib is np else torch.cat(list(locals_), 1)
    # blocks is [N2, N1] with X[k1 + N1*k2] at [k2, k1]
    return blocks.reshape(-1)


def exchange(send, recv, group=None):
    """The all-to-all of one plane: segment r of this rank's send buffer goes
    to slot (this rank) of rank r's receive buffer."""
    import torch.distributed as dist
    with _ffi.nvtx_range("sfft_dist_all_to_all"):
        dist.all_to_all_single(recv, send, group=group)
    return recv


def fft_dist(x_re, x_im, plan=None, *, m=None, inverse=False, group=None, phase_fn=None, exchange_fn=None):
    """One sharded transform: this rank's local input block -> local output.

    ``x_re``/``x_im``: this rank's [N1, N2/G] block (``scatter_input``).
    Returns the local output [N2, N1/G] planes (``gather_output`` layout).
    ``phase_fn(phase, xr, xi) -> (yr, yi)`` and ``exchange_fn(send, recv)``
    default to the CUDA phases and the torch.distributed all-to-all.
    """
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if plan is None and phase_fn is None:
        plan = DistPlan(m, world, rank, dtype=x_re.dtype, device=x_re.device)
    if phase_fn is None:
        def phase_fn(ph, xr, xi):
            yr = torch.empty(plan.local_elems, dtype=xr.dtype, device=xr.device)
            yi = torch.empty_like(yr)
            return plan.phase(ph, xr.contiguous().reshape(-1), xi.contiguous().reshape(-1), yr, yi,
                              inverse=inverse)
    if exchange_fn is None:
        exchange_fn = lambda s, r: exchange(s, r, group)   # noqa: E731
    sr, si = phase_fn(0, x_re, x_im)
    rr, ri = torch.empty_like(sr), torch.empty_like(si)
    exchange_fn(sr, rr)
    exchange_fn(si, ri)
    yr, yi = phase_fn(1, rr, ri)
    l1 = m // 2 if plan is None else plan.l1
    mm = m if plan is None else plan.m
    shape = (1 << (mm - l1), (1 << l1) // world)
    return yr.reshape(shape), yi.reshape(shape)
