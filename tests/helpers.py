"""Shared test helpers: oracle-side network evaluation and comparisons."""

import numpy as np

from oracle import voxmesh_oracle as O


def node_tuples(graph):
    return [(n.id, n.op, n.inputs, n.k, n.c_in, n.c_out) for n in graph.nodes]


def oracle_step(graph, params, x, oh, dtype=np.float64, round_bf16=False):
    """Dense oracle forward/backward in ``dtype``; returns (probs, stats, grads)."""
    cast = (lambda a: O.bf16_round(a).astype(dtype)) if round_bf16 else (lambda a: np.asarray(a, dtype))
    p = {k: {"kernel": cast(v["kernel"]), "bias": np.asarray(v["bias"], dtype)} for k, v in params.items()}
    nodes = node_tuples(graph)
    probs, tape, _ = O.oracle_forward(nodes, p, cast(x))
    ohd = np.asarray(oh, dtype)
    stats = O.loss_stats(probs, ohd)
    total = int(np.prod(x.shape[:4]))
    dprobs = O.loss_grad(probs, ohd, stats, total)
    grads, _ = O.oracle_backward(nodes, p, tape, dprobs)
    return probs, stats, grads, total


def rel_l2(a, b):
    return O.rel_l2(a, b)


class TorchPacker:
    """Test-only stand-in for the CUDA box kernels (tensor slicing), so the halo
    protocol and its transports can be exercised on CPU."""

    @staticmethod
    def _sl(lo5, ext5):
        return tuple(slice(int(a), int(a) + int(e)) for a, e in zip(lo5, ext5))

    def pack(self, buf5, lo5, ext5):
        return buf5[self._sl(lo5, ext5)].clone().contiguous()

    def unpack(self, buf5, lo5, ext5, t):
        buf5[self._sl(lo5, ext5)] = t.reshape(tuple(int(e) for e in ext5))

    def unpack_add(self, buf5, lo5, ext5, t):
        buf5[self._sl(lo5, ext5)] += t.reshape(tuple(int(e) for e in ext5))

    def zero(self, buf5, lo5, ext5):
        buf5[self._sl(lo5, ext5)] = 0
