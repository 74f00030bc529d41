"""CPU oracle for the spatially-partitioned 3D U-Net train step (TEST INFRASTRUCTURE).

This module is a numpy restatement of the reference ``voxmesh`` 0.1.0 algorithms
(``/root/reference/pkg/src/voxmesh``) on the hot path named by BASELINE.json's
north star.  It exists only as the *checker*: ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import it; the
product package ``paper_1909_03108_b200`` never does (its ops fail loudly when the
CUDA library is missing).

Parity of this restatement is PINNED against golden vectors produced by running
the reference itself in the build container (``tests/golden/make_golden.py`` ->
``tests/golden/voxmesh_golden.npz``), and against the hand-checked known answers of
the reference's own tests (``pkg/tests/test_halo.py:54-64``, ``:163-171``,
``test_ops.py:60-71``, ``test_training.py:58-86``, ``test_unet.py:114-120``).

Every function cites the reference file:line it restates.  Arithmetic is done in
the dtype of the inputs; pass float64 arrays to get the f64 oracle that the
tolerance protocol compares against.
"""

from __future__ import annotations

import itertools
import math

import numpy as np

SPATIAL = ("x", "y", "z")
DICE_EPS = 1e-6  # training.py:39


# ---------------------------------------------------------------------------
# Mesh topology (mesh.py:261-276, :78-87) and block geometry (sharding.py:123-143)
# ---------------------------------------------------------------------------


def mesh_coords(shape):
    """Lexicographic rank -> coordinate map (mesh.py:275-276)."""
    return list(itertools.product(*[range(s) for s in shape]))


def neighbor(coord, shape, axis_i, delta):
    """Rank-free neighbor coordinate one step along an axis, None at the edge (mesh.py:78-87)."""
    c = coord[axis_i] + delta
    if c < 0 or c >= shape[axis_i]:
        return None
    return coord[:axis_i] + (c,) + coord[axis_i + 1 :]


def local_slices(dims, layout, axes, coord):
    """Global-index slices of one block (sharding.py:132-143).

    ``dims``: ((name, extent), ...); ``layout``: {dim: axis}; ``axes``: ((name, size), ...).
    """
    axis_index = {a: i for i, (a, _) in enumerate(axes)}
    sizes = dict(axes)
    out = []
    for n, e in dims:
        a = layout.get(n)
        if a is None:
            out.append(slice(0, e))
        else:
            k = e // sizes[a]
            c = coord[axis_index[a]]
            out.append(slice(c * k, (c + 1) * k))
    return tuple(out)


def shard_blocks(x, dims, layout, axes):
    """Bit-exact block cut, one per coordinate in rank order (sharding.py:189-201)."""
    shape = tuple(s for _, s in axes)
    return [np.ascontiguousarray(x[local_slices(dims, layout, axes, c)]) for c in mesh_coords(shape)]


def gather_blocks(blocks, dims, layout, axes, dtype):
    """Reassemble the global tensor bitwise (sharding.py:204-209)."""
    out = np.empty(tuple(e for _, e in dims), dtype=dtype)
    shape = tuple(s for _, s in axes)
    for c, b in zip(mesh_coords(shape), blocks):
        out[local_slices(dims, layout, axes, c)] = b
    return out


# ---------------------------------------------------------------------------
# Halo exchange (halo.py:109-229), simulated over all blocks of the mesh
# ---------------------------------------------------------------------------


def _slab(a, i, start, stop):
    idx = [slice(None)] * a.ndim
    idx[i] = slice(start, stop)
    return a[tuple(idx)]


def halo_exchange_blocks(blocks, dims, layout, axes, margins):
    """Sequential per-dim exchange with zero fill at the global edge (halo.py:109-155).

    ``margins``: {dim: (lo, hi)}.  Phase i operates on the data padded by phases
    < i, so corners arrive through successive hops exactly as in the reference.
    Returns (padded_blocks, bytes_sent_total).
    """
    shape = tuple(s for _, s in axes)
    coords = mesh_coords(shape)
    rank_of = {c: r for r, c in enumerate(coords)}
    axis_index = {a: i for i, (a, _) in enumerate(axes)}
    data = [b for b in blocks]
    nbytes = 0
    for i, (dname, _) in enumerate(dims):
        lo, hi = margins.get(dname, (0, 0))
        if lo == 0 and hi == 0:
            continue
        axis = layout.get(dname)
        # messages: (src, dst, direction) -> slab   (halo.py:131-134)
        msgs = {}
        for r, c in enumerate(coords):
            cur = data[r].shape[i]
            lo_n = neighbor(c, shape, axis_index[axis], -1) if axis else None
            hi_n = neighbor(c, shape, axis_index[axis], +1) if axis else None
            if lo_n is not None and hi > 0:
                m = np.ascontiguousarray(_slab(data[r], i, 0, hi))
                msgs[(r, rank_of[lo_n], "down")] = m
                nbytes += m.nbytes
            if hi_n is not None and lo > 0:
                m = np.ascontiguousarray(_slab(data[r], i, cur - lo, cur))
                msgs[(r, rank_of[hi_n], "up")] = m
                nbytes += m.nbytes
        new = []
        for r, c in enumerate(coords):
            d = data[r]
            lo_n = neighbor(c, shape, axis_index[axis], -1) if axis else None
            hi_n = neighbor(c, shape, axis_index[axis], +1) if axis else None
            if lo_n is not None and lo > 0:  # halo.py:136-141
                lo_slab = msgs[(rank_of[lo_n], r, "up")]
            else:
                s = list(d.shape)
                s[i] = lo
                lo_slab = np.zeros(s, d.dtype)
            if hi_n is not None and hi > 0:  # halo.py:142-147
                hi_slab = msgs[(rank_of[hi_n], r, "down")]
            else:
                s = list(d.shape)
                s[i] = hi
                hi_slab = np.zeros(s, d.dtype)
            new.append(np.concatenate([lo_slab, d, hi_slab], axis=i))  # halo.py:148
        data = new
    return [d.copy() for d in data], nbytes


def halo_exchange_backward_blocks(grads, dims, layout, axes, margins):
    """Exact adjoint: dims reversed, interior kept, low side added first (halo.py:158-194)."""
    shape = tuple(s for _, s in axes)
    coords = mesh_coords(shape)
    rank_of = {c: r for r, c in enumerate(coords)}
    axis_index = {a: i for i, (a, _) in enumerate(axes)}
    data = [g for g in grads]
    for i, (dname, _) in reversed(list(enumerate(dims))):
        lo, hi = margins.get(dname, (0, 0))
        if lo == 0 and hi == 0:
            continue
        axis = layout.get(dname)
        msgs = {}
        for r, c in enumerate(coords):
            cur = data[r].shape[i]
            core = cur - lo - hi
            lo_n = neighbor(c, shape, axis_index[axis], -1) if axis else None
            hi_n = neighbor(c, shape, axis_index[axis], +1) if axis else None
            if lo_n is not None and lo > 0:  # halo.py:176-177
                msgs[(r, rank_of[lo_n], "down")] = np.ascontiguousarray(_slab(data[r], i, 0, lo))
            if hi_n is not None and hi > 0:  # halo.py:178-179
                msgs[(r, rank_of[hi_n], "up")] = np.ascontiguousarray(
                    _slab(data[r], i, lo + core, cur)
                )
        new = []
        for r, c in enumerate(coords):
            cur = data[r].shape[i]
            core = cur - lo - hi
            lo_n = neighbor(c, shape, axis_index[axis], -1) if axis else None
            hi_n = neighbor(c, shape, axis_index[axis], +1) if axis else None
            out = np.array(_slab(data[r], i, lo, lo + core))  # halo.py:180 (owned copy)
            if lo_n is not None and hi > 0:  # halo.py:181-183
                v = _slab(out, i, 0, hi)
                v += msgs[(rank_of[lo_n], r, "up")]
            if hi_n is not None and lo > 0:  # halo.py:184-186
                v = _slab(out, i, core - lo, core)
                v += msgs[(rank_of[hi_n], r, "down")]
            new.append(out)
        data = new
    return [d.copy() for d in data]


def exchange_byte_count(dims, layout, axes, margins, itemsize, direction="forward"):
    """Analytic bytes of the sequential 3-phase protocol (halo.py:197-229)."""
    shape = tuple(s for _, s in axes)
    sizes = dict(axes)
    axis_index = {a: i for i, (a, _) in enumerate(axes)}
    base = []
    for n, e in dims:
        a = layout.get(n)
        base.append(e // sizes[a] if a else e)
    total = 0
    for coord in mesh_coords(shape):
        cur = list(base)
        for i, (name, _) in enumerate(dims):
            lo, hi = margins.get(name, (0, 0))
            if lo == 0 and hi == 0:
                continue
            axis = layout.get(name)
            if axis is not None and sizes[axis] > 1:
                area = 1
                for j, e in enumerate(cur):
                    if j != i:
                        area *= e
                c = coord[axis_index[axis]]
                down_w, up_w = (hi, lo) if direction == "forward" else (lo, hi)
                if c > 0:
                    total += down_w * area
                if c < sizes[axis] - 1:
                    total += up_w * area
            cur[i] += lo + hi
    return total * itemsize


# ---------------------------------------------------------------------------
# Dense single-device kernels (oracle.py:23-118; ops.py:69-199)
# ---------------------------------------------------------------------------


def conv3d_dense(x, kernel, bias):
    """SAME zero-padded cross-correlation; bias first, taps (dz,dy,dx) row-major (oracle.py:23-42)."""
    k = kernel.shape[0]
    m = (k - 1) // 2
    xp = np.pad(x, ((0, 0), (m, m), (m, m), (m, m), (0, 0)))
    b, zs, ys, xs = x.shape[:4]
    c_in, c_out = kernel.shape[3], kernel.shape[4]
    out = np.empty((b, zs, ys, xs, c_out), dtype=x.dtype)
    out[...] = bias.astype(x.dtype, copy=False)
    flat = out.reshape(-1, c_out)
    for dz in range(k):
        for dy in range(k):
            for dx in range(k):
                win = np.ascontiguousarray(xp[:, dz : dz + zs, dy : dy + ys, dx : dx + xs, :]).reshape(-1, c_in)
                flat += win @ kernel[dz, dy, dx]
    return out


def conv3d_dense_backward(gout, x, kernel):
    """(grad_x, grad_kernel, grad_bias) of the SAME conv (oracle.py:45-76)."""
    k = kernel.shape[0]
    m = (k - 1) // 2
    c_in, c_out = kernel.shape[3], kernel.shape[4]
    b, zs, ys, xs = gout.shape[:4]
    gxp = np.zeros((b, zs + 2 * m, ys + 2 * m, xs + 2 * m, c_in), dtype=gout.dtype)
    gflat = np.ascontiguousarray(gout).reshape(-1, c_out)
    for dz in range(k):
        for dy in range(k):
            for dx in range(k):
                c = gflat @ kernel[dz, dy, dx].T
                gxp[:, dz : dz + zs, dy : dy + ys, dx : dx + xs, :] += c.reshape(b, zs, ys, xs, c_in)
    gx = np.ascontiguousarray(gxp[:, m : m + zs, m : m + ys, m : m + xs, :])
    xp = np.pad(x, ((0, 0), (m, m), (m, m), (m, m), (0, 0)))
    gk = np.zeros(kernel.shape, dtype=gout.dtype)
    gb = np.zeros((c_out,), dtype=gout.dtype)
    for s in range(b):
        gs = np.ascontiguousarray(gout[s]).reshape(-1, c_out)
        for dz in range(k):
            for dy in range(k):
                for dx in range(k):
                    win = np.ascontiguousarray(xp[s, dz : dz + zs, dy : dy + ys, dx : dx + xs, :]).reshape(-1, c_in)
                    gk[dz, dy, dx] += win.T @ gs
        gb += gs.sum(axis=0)
    return gx, gk, gb


def maxpool2_dense(x):
    """2^3 max pool; ties go to the first voxel in (dz,dy,dx) scan order (ops.py:141-156)."""
    b, zs, ys, xs, c = x.shape
    cells = x.reshape(b, zs // 2, 2, ys // 2, 2, xs // 2, 2, c).transpose(0, 1, 3, 5, 2, 4, 6, 7)
    cells = cells.reshape(b, zs // 2, ys // 2, xs // 2, 8, c)
    idx = cells.argmax(axis=4)
    return np.take_along_axis(cells, idx[..., None, :], axis=4)[..., 0, :], idx


def maxpool2_dense_backward(gout, idx, in_shape):
    """Route each cell's gradient to its argmax voxel (ops.py:159-168)."""
    b, zs, ys, xs, c = in_shape
    g = np.zeros((b, zs // 2, ys // 2, xs // 2, 8, c), dtype=gout.dtype)
    np.put_along_axis(g, idx[..., None, :], gout[..., None, :], axis=4)
    return g.reshape(b, zs // 2, ys // 2, xs // 2, 2, 2, 2, c).transpose(0, 1, 4, 2, 5, 3, 6, 7).reshape(in_shape)


def upsample2_dense(x):
    """Nearest x2 (ops.py:171-173)."""
    return np.repeat(np.repeat(np.repeat(x, 2, axis=1), 2, axis=2), 2, axis=3)


def upsample2_dense_backward(gout):
    """Sum each 2^3 cell (ops.py:176-179)."""
    b, zs, ys, xs, c = gout.shape
    return gout.reshape(b, zs // 2, 2, ys // 2, 2, xs // 2, 2, c).sum(axis=(2, 4, 6))


def softmax_dense(x):
    """Stable per-voxel softmax over channels (ops.py:190-194)."""
    m = x.max(axis=-1, keepdims=True)
    e = np.exp(x - m)
    return e / e.sum(axis=-1, keepdims=True)


def softmax_dense_backward(gout, probs):
    """probs * (g - <g, probs>) (ops.py:197-199)."""
    dot = (gout * probs).sum(axis=-1, keepdims=True)
    return probs * (gout - dot)


# ---------------------------------------------------------------------------
# Loss + optimizer (training.py:68-127, :202-219)
# ---------------------------------------------------------------------------


def one_hot(labels, num_classes, dtype=np.float32):
    """training.py:68-69"""
    return np.eye(num_classes, dtype=dtype)[labels]


def loss_stats(probs, onehot, clamp=1e-12):
    """[sum p*g, sum p, sum g] per class + summed NLL, sample by sample (training.py:77-92)."""
    c = probs.shape[-1]
    out = np.zeros(3 * c + 1, dtype=probs.dtype)
    for b in range(probs.shape[0]):
        p = probs[b].reshape(-1, c)
        g = onehot[b].reshape(-1, c)
        out[0:c] += (p * g).sum(axis=0)
        out[c : 2 * c] += p.sum(axis=0)
        out[2 * c : 3 * c] += g.sum(axis=0)
        out[3 * c] += -(np.log(np.maximum(p, clamp)) * g).sum()
    return out


def losses_from_stats(stats, num_classes, total_voxels, dice_classes=(1, 2), w_dice=0.9, w_ce=0.1):
    """(combined, dice, ce) (training.py:95-107)."""
    c = num_classes
    pg, ps, gs = stats[0:c], stats[c : 2 * c], stats[2 * c : 3 * c]
    ratios = [(2.0 * float(pg[k]) + DICE_EPS) / (float(ps[k]) + float(gs[k]) + DICE_EPS) for k in dice_classes]
    dice = 1.0 - sum(ratios) / len(ratios)
    ce = float(stats[3 * c]) / total_voxels
    return w_dice * dice + w_ce * ce, dice, ce


def loss_grad(probs, onehot, stats, total_voxels, dice_classes=(1, 2), w_dice=0.9, w_ce=0.1, clamp=1e-12):
    """dLoss/dprobs from the reduced statistics (training.py:110-127)."""
    c = probs.shape[-1]
    pg, ps, gs = stats[0:c], stats[c : 2 * c], stats[2 * c : 3 * c]
    grad = np.zeros_like(probs)
    nfg = len(dice_classes)
    for k in dice_classes:
        nk = 2.0 * float(pg[k]) + DICE_EPS
        dk = float(ps[k]) + float(gs[k]) + DICE_EPS
        r = nk / dk
        grad[..., k] += (-w_dice / nfg) * ((2.0 * onehot[..., k] - r) / dk)
    pm = np.maximum(probs, clamp)
    grad += (-w_ce / total_voxels) * (onehot / pm) * (probs >= clamp)
    return grad


def sgd_momentum_step(params, moments, grads, lr, momentum, order):
    """v = mu*v + g; p -= lr*v; non-finite layers skipped (training.py:202-219)."""
    skipped = []
    for nid in order:
        gk, gb = grads[nid]
        if not (np.isfinite(gk).all() and np.isfinite(gb).all()):
            skipped.append(nid)
            continue
        for key, g in (("kernel", gk), ("bias", gb)):
            v = moments[nid][key]
            v *= momentum
            v += g
            params[nid][key] -= lr * v
    return skipped


# ---------------------------------------------------------------------------
# U-Net graph restatement (unet.py:93-112, :191-225, :284-299) and dense fwd/bwd
# (oracle.py:126-202)
# ---------------------------------------------------------------------------


def recipe_filters(extent, scale=1.0):
    """Filter ladder of recipe_for_resolution (unet.py:93-112)."""
    exp = int(math.log2(extent))
    n_blocks = max(1, 3 + exp - int(math.log2(64)))
    first = 256 * 64 // extent if extent >= 64 else 256
    return tuple(max(1, round(first * (1 << i) * scale)) for i in range(n_blocks))


def graph_nodes(filters, convs_per_block=4, num_classes=3, in_channels=1, kernel=3):
    """Node list (id, op, inputs, k, c_in, c_out) in execution order (unet.py:191-225)."""
    nodes = []
    prev, c_prev = "input", in_channels
    skips = {}
    n = len(filters)
    for i, f in enumerate(filters):
        for j in range(convs_per_block):
            nodes.append((f"enc{i}_conv{j}", "conv", (prev,), kernel, c_prev, f))
            nodes.append((f"enc{i}_relu{j}", "relu", (f"enc{i}_conv{j}",), 0, f, f))
            prev, c_prev = f"enc{i}_relu{j}", f
        if i < n - 1:
            skips[i] = (prev, c_prev)
            nodes.append((f"enc{i}_pool", "pool", (prev,), 0, f, f))
            prev = f"enc{i}_pool"
    for i in range(n - 2, -1, -1):
        f = filters[i]
        nodes.append((f"dec{i}_up", "up", (prev,), 0, c_prev, c_prev))
        sid, sc = skips[i]
        nodes.append((f"dec{i}_cat", "concat", (f"dec{i}_up", sid), 0, c_prev + sc, c_prev + sc))
        prev, c_prev = f"dec{i}_cat", c_prev + sc
        for j in range(convs_per_block):
            nodes.append((f"dec{i}_conv{j}", "conv", (prev,), kernel, c_prev, f))
            nodes.append((f"dec{i}_relu{j}", "relu", (f"dec{i}_conv{j}",), 0, f, f))
            prev, c_prev = f"dec{i}_relu{j}", f
    nodes.append(("head", "conv", (prev,), 1, c_prev, num_classes))
    nodes.append(("softmax", "softmax", ("head",), 0, num_classes, num_classes))
    return nodes


def init_params(nodes, seed, dtype=np.float32):
    """He-uniform U(+-sqrt(6/fan_in)) drawn in conv-node order from one generator (unet.py:284-299)."""
    rng = np.random.default_rng(seed)
    params = {}
    for nid, op, _, k, ci, co in nodes:
        if op != "conv":
            continue
        bound = math.sqrt(6.0 / (k ** 3 * ci))
        kernel = rng.uniform(-bound, bound, (k, k, k, ci, co))
        params[nid] = {"kernel": kernel.astype(dtype), "bias": np.zeros((co,), dtype=dtype)}
    return params


def oracle_forward(nodes, params, x):
    """Dense forward with tape (oracle.py:126-159)."""
    acts = {"input": x}
    tape = {}
    for nid, op, inputs, k, ci, co in nodes:
        a = acts[inputs[0]]
        if op == "conv":
            out = conv3d_dense(a, params[nid]["kernel"], params[nid]["bias"])
            tape[nid] = a
        elif op == "relu":
            out = np.maximum(a, 0)
            tape[nid] = a
        elif op == "pool":
            out, idx = maxpool2_dense(a)
            tape[nid] = (idx, a.shape)
        elif op == "up":
            out = upsample2_dense(a)
        elif op == "concat":
            out = np.concatenate([a, acts[inputs[1]]], axis=-1)
            tape[nid] = a.shape[-1]
        elif op == "softmax":
            out = softmax_dense(a)
            tape[nid] = out
        else:
            raise ValueError(op)
        acts[nid] = out
    return acts[nodes[-1][0]], tape, acts


def oracle_backward(nodes, params, tape, dout):
    """Dense backward; returns ({conv id: (gk, gb)}, grads of every activation) (oracle.py:162-202)."""
    gacts = {nodes[-1][0]: dout}
    seen = {}

    def acc(nid, g):
        if nid == "input":
            return
        gacts[nid] = gacts[nid] + g if nid in gacts else g

    pgrads = {}
    for nid, op, inputs, k, ci, co in reversed(nodes):
        g = gacts.pop(nid, None)
        if g is None:
            continue
        seen[nid] = g
        if op == "conv":
            x = tape.pop(nid)
            gx, gk, gb = conv3d_dense_backward(g, x, params[nid]["kernel"])
            pgrads[nid] = (gk, gb)
            acc(inputs[0], gx)
        elif op == "relu":
            x = tape.pop(nid)
            acc(inputs[0], np.where(x > 0, g, np.zeros((), dtype=g.dtype)))
        elif op == "pool":
            idx, in_shape = tape.pop(nid)
            acc(inputs[0], maxpool2_dense_backward(g, idx, in_shape))
        elif op == "up":
            acc(inputs[0], upsample2_dense_backward(g))
        elif op == "concat":
            ca = tape.pop(nid)
            acc(inputs[0], np.ascontiguousarray(g[..., :ca]))
            acc(inputs[1], np.ascontiguousarray(g[..., ca:]))
        elif op == "softmax":
            probs = tape.pop(nid)
            acc(inputs[0], softmax_dense_backward(g, probs))
    return pgrads, seen


def train_step(nodes, params, moments, x, onehot, lr=0.003, momentum=0.9, clamp=1e-12):
    """One dense step: fwd -> stats -> loss grad -> bwd -> SGD (training.py:330-343)."""
    probs, tape, _ = oracle_forward(nodes, params, x)
    stats = loss_stats(probs, onehot, clamp)
    total = int(np.prod(x.shape[:4]))
    dprobs = loss_grad(probs, onehot, stats, total, clamp=clamp)
    grads, _ = oracle_backward(nodes, params, tape, dprobs)
    order = tuple(n[0] for n in nodes if n[1] == "conv")
    skipped = sgd_momentum_step(params, moments, grads, lr, momentum, order)
    return losses_from_stats(stats, onehot.shape[-1], total), grads, skipped


# ---------------------------------------------------------------------------
# Synthetic CT-like record (data_io.py:155-184) — the synthetic-input spec
# ---------------------------------------------------------------------------


def _ellipsoid_mask(shape, center, radii):
    grids = np.ogrid[tuple(slice(0, s) for s in shape)]
    acc = np.zeros(shape, dtype=np.float64)
    for g, c, r in zip(grids, center, radii):
        acc = acc + ((g - c) / r) ** 2
    return acc <= 1.0


def synthesize_record(extent, rng):
    """Noise background, +1.0 liver ellipsoid (label 1), +1.5 tumors (label 2) (data_io.py:163-184)."""
    shape = (extent,) * 3
    image = rng.normal(0.0, 0.1, shape)
    center = [extent / 2 + rng.uniform(-extent / 10, extent / 10) for _ in range(3)]
    radii = [rng.uniform(0.30, 0.40) * extent for _ in range(3)]
    liver = _ellipsoid_mask(shape, center, radii)
    labels = np.zeros(shape, dtype=np.uint8)
    labels[liver] = 1
    image = image + 1.0 * liver
    liver_idx = np.argwhere(liver)
    n_tumors = int(rng.integers(1, 4))
    tumor = np.zeros(shape, dtype=bool)
    for _ in range(n_tumors):
        c = liver_idx[rng.integers(len(liver_idx))]
        r = rng.uniform(extent / 16, extent / 8)
        tumor |= _ellipsoid_mask(shape, c, (r, r, r))
    tumor &= liver
    labels[tumor] = 2
    image = image + 1.5 * tumor
    return image.astype(np.float32), labels


def record_for(extent, i, seed=7):
    """Record ``i`` of a synthetic dataset with seed ``seed`` (data_io.py:196)."""
    return synthesize_record(extent, np.random.default_rng(np.random.SeedSequence([int(seed), i])))


# ---------------------------------------------------------------------------
# Helpers for the tolerance protocol
# ---------------------------------------------------------------------------


def bf16_round(a):
    """Round-to-nearest-even to bfloat16, returned as float32 (the GPU storage rounding)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    out = rounded.astype(np.uint32).view(np.float32)
    nan = np.isnan(a)
    if nan.any():
        out = out.copy()
        out[nan] = np.nan
    return out


def rel_l2(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.linalg.norm(ref.ravel())
    return float(np.linalg.norm((got - ref).ravel()) / max(den, 1e-30))
