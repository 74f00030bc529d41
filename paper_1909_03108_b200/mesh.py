"""Device mesh: rank <-> coordinate topology, SPMD dispatch, point-to-point and collectives.

Same API as the reference ``voxmesh/mesh.py`` (DeviceMesh, WorkerContext,
create_mesh; lexicographic rank <-> coord, mesh.py:261-276; +-1 neighbours with
None at the edge, mesh.py:78-87; axis groups sorted by coordinate,
mesh.py:142-157; all_reduce_sum summing in coordinate order, mesh.py:195-233),
with two transports behind it:

``threads``  (single process, the default when torch.distributed is not
             initialised): one worker thread per mesh rank, each with its own
             CUDA stream, all on the current CUDA device unless ``devices=``
             spreads them (payloads that arrive from another device are copied
             to the receiver's device on its stream).  Payloads are
             device tensors handed over FIFO queues together with a CUDA event
             recorded on the sender's stream; the receiver's stream waits on it.
             This is how the multi-rank parity tests run on ONE GPU: every rank
             is a real CUDA stream running the real pack/unpack kernels.
``spmd``     (one process per GPU under torchrun, torch.distributed initialised
             with world_size == worker_count): each process owns its rank; halo
             messages are grouped ``batch_isend_irecv`` (NCCL send/recv over
             NVLink) and reductions are ``all_reduce`` over cached axis groups.
"""

from __future__ import annotations

import itertools
import queue
import threading
import traceback
from dataclasses import dataclass

import numpy as np

from .errors import (
    CollectiveMismatchError,
    DeadlockError,
    MeshConfigError,
    ProtocolError,
    WorkerFailed,
    WorkerShutdown,
)

_STOP = object()


@dataclass(frozen=True)
class MeshAxis:
    name: str
    size: int


def _nbytes(payload):
    if payload is None:
        return 0
    if hasattr(payload, "element_size") and hasattr(payload, "numel"):
        return int(payload.element_size() * payload.numel())
    if isinstance(payload, np.ndarray):
        return int(payload.nbytes)
    if isinstance(payload, (tuple, list)):
        return sum(_nbytes(p) for p in payload)
    return 0


def _torch():
    import torch

    return torch


class WorkerContext:
    """Per-rank view: coordinate, device + stream, transport, counters, persistent store."""

    def __init__(self, mesh, rank):
        self.mesh = mesh
        self.rank = rank
        self.coord = mesh.coords[rank]
        self.store = {}
        self.counters = {"p2p_bytes": 0, "p2p_msgs": 0, "coll_bytes": 0}
        self.device = mesh.device_of(rank)
        self._stream = None

    @property
    def stream(self):
        torch = _torch()
        if self._stream is None and self.device.type == "cuda":
            self._stream = torch.cuda.Stream(device=self.device)
        return self._stream

    # ---- topology ---------------------------------------------------------
    def axis_size(self, axis):
        return self.mesh.axis_size(axis)

    def axis_coord(self, axis):
        return self.coord[self.mesh.axis_index[axis]]

    def neighbor(self, axis, delta):
        if delta not in (-1, 1):
            raise ProtocolError(f"neighbor step must be +/-1, got {delta}")
        i = self.mesh.axis_index[axis]
        c = self.coord[i] + delta
        if not 0 <= c < self.mesh.axes[i].size:
            return None
        return self.mesh.rank_of[self.coord[:i] + (c,) + self.coord[i + 1 :]]

    def _neighbor_ranks(self):
        out = set()
        for ax in self.mesh.axes:
            for d in (-1, 1):
                r = self.neighbor(ax.name, d)
                if r is not None:
                    out.add(r)
        return out

    def group(self, axes=None):
        if axes is None:
            axes = [a.name for a in self.mesh.axes]
        elif isinstance(axes, str):
            axes = [axes]
        idx = []
        for a in axes:
            if a not in self.mesh.axis_index:
                raise MeshConfigError(f"unknown mesh axis {a!r}")
            idx.append(self.mesh.axis_index[a])
        ranges = [range(ax.size) if i in idx else (self.coord[i],) for i, ax in enumerate(self.mesh.axes)]
        return [self.mesh.rank_of[c] for c in itertools.product(*ranges)]

    # ---- point to point -----------------------------------------------------
    def send(self, dst, payload, tag):
        if dst not in self._neighbor_ranks():
            raise ProtocolError(f"{self.coord} -> {self.mesh.coords[dst]}: not mesh neighbors")
        self.counters["p2p_bytes"] += _nbytes(payload)
        self.counters["p2p_msgs"] += 1
        self.mesh._transport_send(self, dst, payload, tag)

    def recv(self, src, tag, like=None):
        return self.mesh._transport_recv(self, src, tag, like)

    def exchange(self, sends, recvs):
        """Grouped neighbour exchange: ``sends`` = [(dst, tensor, tag)], ``recvs`` =
        [(src, like_tensor, tag)] -> received tensors (NCCL group in spmd mode)."""
        for dst, t, _ in sends:
            if dst not in self._neighbor_ranks():
                raise ProtocolError(f"{self.coord} -> {self.mesh.coords[dst]}: not mesh neighbors")
            self.counters["p2p_bytes"] += _nbytes(t)
            self.counters["p2p_msgs"] += 1
        return self.mesh._transport_exchange(self, sends, recvs)

    # ---- collectives ----------------------------------------------------------
    def barrier(self, axes=None, tag="barrier"):
        self.mesh._barrier(self, axes, tag)

    def all_reduce_sum(self, local, axes=None, tag="allreduce"):
        """Element-wise sum over the axis group; identical result on every member."""
        return self.mesh._all_reduce(self, local, axes, tag)


class DeviceMesh:
    """A grid of devices; ranks enumerate coordinates lexicographically."""

    def __init__(self, axes, timeout=30.0, backend="auto", devices=None):
        axes = [MeshAxis(str(n), int(s)) for n, s in axes]
        if not axes:
            raise MeshConfigError("mesh needs at least one axis")
        names = [a.name for a in axes]
        if len(set(names)) != len(names):
            raise MeshConfigError(f"duplicate axis names in {names}")
        for a in axes:
            if a.size < 1:
                raise MeshConfigError(f"axis {a.name!r} has non-positive size {a.size}")
        self.axes = tuple(axes)
        self.axis_index = {a.name: i for i, a in enumerate(axes)}
        self.shape = tuple(a.size for a in axes)
        self.worker_count = int(np.prod(self.shape))
        self.coords = list(itertools.product(*[range(s) for s in self.shape]))
        self.rank_of = {c: r for r, c in enumerate(self.coords)}
        self.timeout = float(timeout)
        self._devices = devices
        self._closed = False
        self._broken = threading.Event()

        import torch.distributed as dist

        spmd_ok = dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
        if backend == "auto":
            backend = "spmd" if spmd_ok else "threads"
        if backend == "spmd":
            if not spmd_ok:
                raise MeshConfigError("spmd backend needs an initialised torch.distributed group")
            if dist.get_world_size() != self.worker_count:
                raise MeshConfigError(
                    f"mesh has {self.worker_count} workers but the process group has "
                    f"{dist.get_world_size()} ranks"
                )
            self.local_ranks = [dist.get_rank()]
        elif backend == "threads":
            self.local_ranks = list(range(self.worker_count))
        else:
            raise MeshConfigError(f"unknown backend {backend!r}")
        self.backend = backend
        self._contexts = {r: WorkerContext(self, r) for r in self.local_ranks}
        self._groups = {}
        if backend == "threads":
            self._channels = {}
            self._chan_lock = threading.Lock()
            self._cmd = {r: queue.Queue() for r in self.local_ranks}
            self._done = queue.Queue()
            self._job = itertools.count()
            self._threads = [
                threading.Thread(target=self._loop, args=(r,), name=f"mesh-{self.coords[r]}", daemon=True)
                for r in self.local_ranks
            ]
            for t in self._threads:
                t.start()
            self.run(lambda ctx: ctx.barrier())

    # ---- placement ------------------------------------------------------------
    def device_of(self, rank):
        torch = _torch()
        if self._devices is not None:
            return torch.device(self._devices[rank % len(self._devices)])
        if not torch.cuda.is_available():
            return torch.device("cpu")
        # spmd: this process's device; threads: every rank on the current device (the
        # single-GPU parity transport) unless devices= spreads them explicitly
        return torch.device("cuda", torch.cuda.current_device())

    def context(self, rank):
        return self._contexts[rank]

    # ---- driver API -------------------------------------------------------------
    def run(self, fn, *args, per_worker=None):
        """Execute ``fn(ctx, *args, *per_worker[rank])`` on every local rank; results by rank."""
        if self._closed:
            raise ProtocolError("mesh is shut down")
        if self._broken.is_set():
            raise ProtocolError("mesh is broken after an earlier failure")
        results = [None] * self.worker_count
        if self.backend == "spmd":
            r = self.local_ranks[0]
            extra = tuple(pw[r] for pw in per_worker) if per_worker else ()
            ctx = self._contexts[r]
            try:
                results[r] = self._call(ctx, fn, args + extra)
            except WorkerShutdown:
                raise
            except Exception as e:  # noqa: BLE001
                raise WorkerFailed(ctx.coord, f"{e}\n{traceback.format_exc()}") from e
            return results
        job = next(self._job)
        for r in self.local_ranks:
            extra = tuple(pw[r] for pw in per_worker) if per_worker else ()
            self._cmd[r].put((job, fn, args + extra))
        first = None
        for _ in self.local_ranks:
            jid, rank, status, payload = self._done.get()
            if status == "ok":
                results[rank] = payload
            elif status == "error" and first is None:
                first = (rank, payload)
                self._poison()
        if first is not None:
            rank, (exc, tb) = first
            raise WorkerFailed(self.coords[rank], f"{exc}\n{tb}") from exc
        return results

    def _call(self, ctx, fn, args):
        torch = _torch()
        if ctx.device.type == "cuda":
            with torch.cuda.device(ctx.device), torch.cuda.stream(ctx.stream):
                out = fn(ctx, *args)
            return out
        return fn(ctx, *args)

    def synchronize(self):
        """Wait for all work queued on every local rank's stream."""
        torch = _torch()
        for ctx in self._contexts.values():
            if ctx.device.type == "cuda":
                ctx.stream.synchronize()

    def shutdown(self):
        if self._closed:
            return
        self._closed = True
        if self.backend == "threads":
            for r in self.local_ranks:
                self._cmd[r].put(_STOP)
            for t in self._threads:
                t.join(timeout=self.timeout)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.shutdown()
        return False

    def axis_size(self, name):
        if name not in self.axis_index:
            raise MeshConfigError(f"unknown mesh axis {name!r}")
        return self.axes[self.axis_index[name]].size

    def describe(self):
        return ",".join(f"{a.name}={a.size}" for a in self.axes)

    # ---- threads backend internals ------------------------------------------------
    def _loop(self, rank):
        ctx = self._contexts[rank]
        while True:
            item = self._cmd[rank].get()
            if item is _STOP:
                return
            job, fn, args = item
            try:
                out = self._call(ctx, fn, args)
            except WorkerShutdown as e:
                self._done.put((job, rank, "shutdown", e))
            except BaseException as e:  # noqa: BLE001
                self._done.put((job, rank, "error", (e, traceback.format_exc())))
            else:
                self._done.put((job, rank, "ok", out))

    def _chan(self, src, dst):
        key = (src, dst)
        q = self._channels.get(key)
        if q is None:
            with self._chan_lock:
                q = self._channels.setdefault(key, queue.Queue())
                if self._broken.is_set():
                    q.put(_STOP)
        return q

    def _poison(self):
        self._broken.set()
        with self._chan_lock:
            for q in self._channels.values():
                q.put(_STOP)

    def _get(self, ctx, src, timeout=None):
        if self._broken.is_set():
            raise WorkerShutdown("mesh is shutting down")
        try:
            item = self._chan(src, ctx.rank).get(timeout=self.timeout if timeout is None else timeout)
        except queue.Empty:
            raise DeadlockError(
                f"{ctx.coord} timed out after {self.timeout}s waiting for a message from "
                f"{self.coords[src]}"
            ) from None
        if item is _STOP:
            raise WorkerShutdown("mesh is shutting down")
        return item

    def _put(self, ctx, dst, payload, tag):
        torch = _torch()
        ev = None
        if ctx.device.type == "cuda":
            # recorded on the stream the payload was produced on (the rank's stream, or a
            # comm stream the caller made current)
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(ctx.device))
        self._chan(ctx.rank, dst).put((tag, payload, ev))

    def _take(self, ctx, src, tag, timeout=None):
        got, payload, ev = self._get(ctx, src, timeout)
        if got != tag:
            raise ProtocolError(f"{ctx.coord} expected tag {tag!r} from {self.coords[src]}, got {got!r}")
        if ev is not None and ctx.device.type == "cuda":
            cur = _torch().cuda.current_stream(ctx.device)
            cur.wait_event(ev)
            if hasattr(payload, "record_stream") and getattr(payload, "is_cuda", False):
                payload.record_stream(cur)
                if payload.device != ctx.device:  # a rank on another GPU: copy in on our stream
                    payload = payload.to(ctx.device, non_blocking=True)
        return payload

    # ---- transport ------------------------------------------------------------------
    def _transport_send(self, ctx, dst, payload, tag):
        if self.backend == "threads":
            self._put(ctx, dst, payload, tag)
        else:
            import torch.distributed as dist

            ctx.store.setdefault("_pending", []).append(dist.isend(payload.contiguous(), dst))

    def _transport_recv(self, ctx, src, tag, like):
        if self.backend == "threads":
            return self._take(ctx, src, tag)
        import torch.distributed as dist

        if like is None:
            raise ProtocolError("spmd recv needs a template tensor (shape/dtype)")
        buf = _torch().empty_like(like)
        dist.recv(buf, src)
        return buf

    def _transport_exchange(self, ctx, sends, recvs):
        if self.backend == "threads":
            for dst, t, tag in sends:
                self._put(ctx, dst, t, tag)
            return [self._take(ctx, src, tag) for src, _, tag in recvs]
        import torch.distributed as dist

        torch = _torch()
        bufs = [torch.empty_like(like) for _, like, _ in recvs]
        ops = [dist.P2POp(dist.isend, t, dst) for dst, t, _ in sends]
        ops += [dist.P2POp(dist.irecv, b, src) for (src, _, _), b in zip(recvs, bufs)]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return bufs

    # ---- collectives ------------------------------------------------------------------
    def _pg(self, ctx, axes):
        """torch.distributed subgroup of the ranks that vary along ``axes`` (cached)."""
        import torch.distributed as dist

        key = tuple(sorted(axes)) if axes is not None else None
        if key in self._groups:
            return self._groups[key]
        if axes is None or len(ctx.group(axes)) == self.worker_count:
            self._groups[key] = None
            return None
        # every process must create every subgroup in the same order
        idx = [self.axis_index[a] for a in ([axes] if isinstance(axes, str) else axes)]
        fixed = [i for i in range(len(self.axes)) if i not in idx]
        mine = None
        for combo in itertools.product(*[range(self.axes[i].size) for i in fixed]):
            members = sorted(
                r for r, c in enumerate(self.coords) if all(c[i] == v for i, v in zip(fixed, combo))
            )
            g = dist.new_group(members)
            if ctx.rank in members:
                mine = g
        self._groups[key] = mine
        return mine

    def _barrier(self, ctx, axes, tag):
        group = ctx.group(axes)
        if len(group) == 1:
            return
        if self.backend == "spmd":
            import torch.distributed as dist

            dist.barrier(group=self._pg(ctx, axes))
            return
        leader = group[0]
        if ctx.rank == leader:
            for r in group[1:]:
                self._take(ctx, r, (tag, "arrive"))
            for r in group[1:]:
                self._put(ctx, r, None, (tag, "release"))
        else:
            self._put(ctx, leader, None, (tag, "arrive"))
            self._take(ctx, leader, (tag, "release"), timeout=self.timeout * (len(group) + 1))

    def _all_reduce(self, ctx, local, axes, tag):
        torch = _torch()
        group = ctx.group(axes)
        is_np = isinstance(local, np.ndarray) or np.isscalar(local)
        if is_np:
            local = np.asarray(local)
        if len(group) == 1:
            return local
        if self.backend == "spmd":
            import torch.distributed as dist

            t = torch.as_tensor(local).to(ctx.device) if is_np else local
            t = t.clone()
            ctx.counters["coll_bytes"] += _nbytes(t)
            dist.all_reduce(t, group=self._pg(ctx, axes))
            return t.cpu().numpy() if is_np else t
        leader = group[0]
        if ctx.rank == leader:
            parts = [local] + [self._take(ctx, r, (tag, "part")) for r in group[1:]]
            bad = [
                (self.coords[group[i]], tuple(p.shape), p.dtype)
                for i, p in enumerate(parts)
                if tuple(p.shape) != tuple(local.shape) or p.dtype != local.dtype
            ]
            if bad:
                err = CollectiveMismatchError(
                    f"all_reduce_sum over {axes or 'all axes'}: expected {tuple(local.shape)} "
                    f"{local.dtype}, got {bad}"
                )
                for r in group[1:]:
                    self._put(ctx, r, err, (tag, "result"))
                raise err
            acc = parts[0].copy() if is_np else parts[0].clone()
            for p in parts[1:]:  # coordinate order, mesh.py:223-225
                acc += p
            for r in group[1:]:
                ctx.counters["coll_bytes"] += _nbytes(acc)
                self._put(ctx, r, acc.copy() if is_np else acc.clone(), (tag, "result"))
            return acc
        ctx.counters["coll_bytes"] += _nbytes(local)
        self._put(ctx, leader, local, (tag, "part"))
        res = self._take(ctx, leader, (tag, "result"))
        if isinstance(res, Exception):
            raise res
        return res


def create_mesh(axes, timeout=30.0, backend="auto", devices=None):
    """Build a DeviceMesh from ``[(axis_name, size), ...]``."""
    return DeviceMesh(axes, timeout=timeout, backend=backend, devices=devices)
