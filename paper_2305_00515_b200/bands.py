"""Row-band partition of one image across ranks (BASELINE config C5).

The reference has no multi-device path; SURVEY.md section 8e specifies it:
rank k of N owns input rows [k*H/N, (k+1)*H/N) and needs the 2 rows above
and the 2 rows below its band (the 2r = 4-row vertical halo of the 5x5
stencil).  Output rows never overlap, so no gather is needed.

Halo transports:

* ``"peer"`` (default on B200): every rank exports its band buffer with CUDA
  IPC (sobel5_ipc_export), maps its neighbours' buffers once, and ONE kernel
  (sobel5_launch_band) reads the neighbour rows over NVLink/NVSwitch while it
  streams its own band: the exchange is fused into the compute, no copy and
  no collective on the data path.  Cross-process ordering is carried by
  stream-ordered flags in a shared host page every rank maps (step
  counters, cuStreamWriteValue32 / cuStreamWaitValue32 through
  sobel5_stream_write_u32 / _wait_u32), without a host barrier per step:
  ``ready[k] = s`` once rank k's input for step s is on its stream, the band
  kernel waits for ``ready[k-1], ready[k+1] >= s``, then ``done[k] = s``, and
  the stream waits for ``done[k-1], done[k+1] >= s`` before anything the
  caller enqueues next (the next step's input) can overwrite rows a
  neighbour is still reading.
* ``"nccl"`` / ``"gloo"``: the 2-row halos are exchanged with
  torch.distributed point-to-point ops (batched isend/irecv).  The interior
  rows, which need no halo, are launched first so the exchange overlaps them;
  two 2-row seam launches follow.  ``"gloo"`` stages through host memory and
  exists so the partition logic runs in CPU-only multi-process tests.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _abi, api

HALO = 2  # rows above / below a band (radius of the 5x5 operator)


@dataclass(frozen=True)
class BandPlan:
    """Which rows rank `rank` of `world` owns and computes."""

    rank: int
    world: int
    width: int
    height: int
    r0: int          # first input row of the band
    r1: int          # one past the last input row
    has_top: bool    # needs rows r0-2, r0-1 from rank-1
    has_bot: bool    # needs rows r1, r1+1 from rank+1
    c0: int          # first centre row computed here (image coordinates)
    c1: int          # one past the last centre row

    @property
    def body_rows(self) -> int:
        return self.r1 - self.r0

    @property
    def out_rows(self) -> int:
        return self.c1 - self.c0

    @property
    def out_row0(self) -> int:
        """Row of the full (W-4)x(H-4) output where this band's rows start."""
        return self.c0 - HALO


def plan_bands(width: int, height: int, world: int, rank: int) -> BandPlan:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if width < 5 or height < 5:
        raise api.ImageTooSmall(f"streaming filter needs at least 5x5, got {width}x{height}")
    if height < 4 * world:
        raise api.DimMismatch(f"{height} rows cannot be split into {world} bands of >= 4 rows")
    r0 = rank * height // world
    r1 = (rank + 1) * height // world
    c0, c1 = max(r0, HALO), min(r1, height - HALO)
    return BandPlan(rank, world, width, height, r0, r1, rank > 0, rank < world - 1, c0, c1)


def _row_ptr(t, row: int, pitch: int) -> int:
    return t.data_ptr() + row * pitch


class RowBandPartition:
    """Runs the fused kernel on this rank's band of a row-partitioned image.

    ``body`` is this rank's band, a (body_rows, pitch) uint8 device tensor.
    """

    def __init__(self, plan: BandPlan, body, pitch: int, transport: str = "peer", group=None):
        import torch.distributed as dist
        self.plan, self.body, self.pitch = plan, body, pitch
        self.transport, self.group = transport, group
        self._peer = {}  # rank -> imported pointer
        self._dist = dist
        self._flags = None  # (mmap, host address, device address) of the shared flag page
        self._step = 0
        if transport not in ("peer", "nccl", "gloo"):
            raise ValueError(transport)
        if plan.world > 1 and transport == "peer":
            self._map_neighbours()
            self._map_flags()

    # ---- peer mapping -----------------------------------------------------------
    def _map_neighbours(self):
        L = _abi.load()
        h = _abi.IpcHandle()
        api.check(L.sobel5_ipc_export(self.body.data_ptr(), C.byref(h)), "sobel5_ipc_export")
        mine = (bytes(h.bytes), int(h.offset))
        handles = [None] * self.plan.world
        self._dist.all_gather_object(handles, mine, group=self.group)
        for nb in (self.plan.rank - 1, self.plan.rank + 1):
            if 0 <= nb < self.plan.world:
                hh = _abi.IpcHandle()
                hh.bytes[:] = list(handles[nb][0])
                hh.offset = handles[nb][1]
                p = C.c_void_p()
                api.check(L.sobel5_ipc_import(C.byref(hh), C.byref(p)), "sobel5_ipc_import")
                self._peer[nb] = p.value
        self._dist.barrier(group=self.group)

    # ---- shared flag page (cross-process stream ordering) ----------------------
    _FLAG_BYTES = 4096
    _DONE = 256  # byte offset of done[]; ready[] starts at 0 (uint32 per rank)

    def _map_flags(self):
        import mmap
        import os
        import uuid
        L = _abi.load()
        name = [f"/dev/shm/sobel5_bands_{uuid.uuid4().hex}" if self.plan.rank == 0 else None]
        self._dist.broadcast_object_list(name, src=0, group=self.group)
        path = name[0]
        if self.plan.rank == 0:
            with open(path, "wb") as f:
                f.write(bytes(self._FLAG_BYTES))
        self._dist.barrier(group=self.group)
        fd = os.open(path, os.O_RDWR)
        try:
            mm = mmap.mmap(fd, self._FLAG_BYTES)
        finally:
            os.close(fd)
        self._dist.barrier(group=self.group)
        if self.plan.rank == 0:
            os.unlink(path)  # every rank holds the mapping; nothing left behind
        host = C.addressof(C.c_char.from_buffer(mm))
        dev = C.c_void_p()
        api.check(L.sobel5_host_register(host, self._FLAG_BYTES, C.byref(dev)),
                  "sobel5_host_register")
        self._flags = (mm, host, dev.value)

    def _flag(self, which: int, rank: int) -> int:
        return self._flags[2] + which + 4 * rank

    def close(self):
        L = _abi.load()
        for p in self._peer.values():
            L.sobel5_ipc_release(p)
        self._peer = {}
        if self._flags is not None:
            mm, host, _ = self._flags
            L.sobel5_host_unregister(host)
            self._flags = None
            try:
                mm.close()
            except BufferError:  # a ctypes view still alive; the OS unmaps at exit
                pass

    # ---- halo exchange through torch.distributed ---------------------------------
    def exchange(self):
        """Returns (top, bot) halo tensors of shape (2, pitch) (None at the
        image edges) received from the neighbours."""
        import torch
        dist, p = self._dist, self.plan
        stage = self.transport == "gloo"
        dev = "cpu" if stage else self.body.device

        def out(rows):
            t = rows.contiguous()
            return t.cpu() if stage else t

        top = torch.empty((HALO, self.pitch), dtype=torch.uint8, device=dev) if p.has_top else None
        bot = torch.empty((HALO, self.pitch), dtype=torch.uint8, device=dev) if p.has_bot else None
        ops = []
        if p.has_top:
            ops.append(dist.P2POp(dist.isend, out(self.body[:HALO]), p.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, top, p.rank - 1, self.group))
        if p.has_bot:
            ops.append(dist.P2POp(dist.isend, out(self.body[-HALO:]), p.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, bot, p.rank + 1, self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        if stage:
            top = top.to(self.body.device) if top is not None else None
            bot = bot.to(self.body.device) if bot is not None else None
        return top, bot

    # ---- compute --------------------------------------------------------------------
    def run(self, taps, planes: dict, out_pitch: int, prefetch: int = 1, stream=None):
        """Writes this rank's plan.out_rows output rows into ``planes``
        (tensors of shape (>= out_rows, out_pitch))."""
        p = self.plan
        if p.world == 1:
            api.launch(self.body, self.pitch, p.width, p.height, taps, prefetch, planes, out_pitch,
                       stream=stream)
            return
        if self.transport == "peer":
            import torch
            L = _abi.load()
            sp = stream if stream is not None else torch.cuda.current_stream().cuda_stream
            self._step = s = (self._step + 1) & 0xFFFFFFFF
            nbrs = [r for r, has in ((p.rank - 1, p.has_top), (p.rank + 1, p.has_bot)) if has]

            def flag_op(fn, which, rank):
                api.check(fn(self._flag(which, rank), s, sp), fn.__name__)

            flag_op(L.sobel5_stream_write_u32, 0, p.rank)  # my rows for step s are in place
            for r in nbrs:
                flag_op(L.sobel5_stream_wait_u32, 0, r)  # neighbours' rows too
            top = _row_ptr_int(self._peer.get(p.rank - 1), self._prev_rows() - HALO, self.pitch) \
                if p.has_top else None
            bot = self._peer.get(p.rank + 1) if p.has_bot else None
            api.launch_band(top, self.body, bot, self.pitch, p.width, p.body_rows, taps, prefetch,
                            planes, out_pitch, stream=sp)
            flag_op(L.sobel5_stream_write_u32, self._DONE, p.rank)  # done reading my halos
            for r in nbrs:  # later writes to my rows wait for the neighbours' reads
                flag_op(L.sobel5_stream_wait_u32, self._DONE, r)
            return
        import torch
        # torch.distributed orders its P2P ops and copies against the CURRENT
        # stream: make that the caller's stream for the whole exchange
        ext = torch.cuda.ExternalStream(stream) if stream is not None else None
        with torch.cuda.stream(ext) if ext is not None else _nullcontext():
            self._run_exchange(taps, planes, out_pitch, prefetch, stream)

    def _run_exchange(self, taps, planes, out_pitch, prefetch, stream):
        p = self.plan
        # interior first (no halo needed), overlapping the exchange
        top_rows = HALO if p.has_top else 0
        interior = p.body_rows - 4
        if interior > 0:
            api.launch_band(None, self.body, None, self.pitch, p.width, p.body_rows, taps, prefetch,
                            _offset_planes(planes, top_rows, out_pitch), out_pitch, stream=stream)
        top, bot = self.exchange()
        if p.has_top:  # centres r0, r0+1 from [top; rows r0..r0+3]
            api.launch_band(top, self.body, None, self.pitch, p.width, 4, taps, prefetch, planes,
                            out_pitch, stream=stream)
        if p.has_bot:  # centres r1-2, r1-1 from [rows r1-4..r1-1; bot]
            tail = self.body[p.body_rows - 4:]
            api.launch_band(None, tail, bot, self.pitch, p.width, 4, taps, prefetch,
                            _offset_planes(planes, p.out_rows - HALO, out_pitch), out_pitch,
                            stream=stream)

    def _prev_rows(self) -> int:
        prev = plan_bands(self.plan.width, self.plan.height, self.plan.world, self.plan.rank - 1)
        return prev.body_rows


class _nullcontext:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


def _row_ptr_int(base: int | None, row: int, pitch: int) -> int | None:
    return None if base is None else base + row * pitch


class _View:
    """A plane pointer offset by whole rows (what launch_band writes into)."""

    def __init__(self, t, off_elems: int):
        self._p = t.data_ptr() + off_elems * t.element_size()

    def data_ptr(self):
        return self._p


def _offset_planes(planes: dict, rows: int, pitch: int) -> dict:
    return {k: _View(v, rows * pitch) for k, v in planes.items()}
