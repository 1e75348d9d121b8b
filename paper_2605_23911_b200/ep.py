"""Expert-parallel MoE layer (DeepSeek-V3 across the GPUs of one box).

The reference has no multi-GPU path (``SPEC.md:8``; ``PAPER.md:430`` item 6).
SURVEY.md §8e specifies the partition used here:

* expert ``e`` lives on rank ``owner(e)`` — contiguous blocks of ``E/n``
  experts (uneven blocks allowed);
* tokens are sharded ``B/n`` per rank; the router weight is replicated, and
  each rank routes its own tokens (rows are independent, so local routing is
  bit-identical to global routing);
* steps: local route → per-expert counts all-to-all → dispatch all-to-all
  (bf16 rows, already expert-major per destination because the local
  permutation is the reference's stable expert-major order) → reorder to
  expert-major across sources → local expert FFN → reorder back → combine
  all-to-all (fp32 rows) → home-rank combine in ascending slot order.

The output is bitwise identical to the single-GPU layer: every row's expert
output is computed by the same kernels with the same K order regardless of
which other rows share its tile, and the home-rank combine runs the
reference's ``out += w_j * g_j`` order (``pipeline.py:396-399``).

Two transports.  ``transport="p2p"`` (``PeerExchange``): the exchanges run
over peer memory in libmoe_b200.so (``csrc/ep_p2p.cuh``: rows written
straight into the owners' buffers, outputs straight back, device-side epoch
flags), with no host synchronisation; the forward is graph-capturable.
``transport="collective"``: ``torch.distributed`` all-to-alls (NCCL on
GPUs), whose one host synchronisation per forward is the counts exchange
that sizes them.  All row compute runs in libmoe_b200.so through ``CudaOps``;
the collective path's host logic is written against a small ops interface so
it can be exercised on CPU with gloo in the tests.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .types import GATING_CODE, ExpertWeights, Gating, ModelConfig


def expert_ranges(num_experts: int, world: int):
    """Contiguous expert blocks: rank r owns [lo_r, hi_r)  (owner(e) = floor(e*n/E))."""
    bounds = [(r * num_experts + world - 1) // world for r in range(world + 1)]
    # owner(e) = floor(e * n / E)  <=>  e in [ceil(r*E/n), ceil((r+1)*E/n))
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def source_major_to_expert_major(recv_counts: np.ndarray) -> np.ndarray:
    """Row order fix-up for the dispatch all-to-all.

    ``recv_counts[src, e]`` rows arrive source-major (src ascending, expert
    ascending within a source).  Returns ``idx`` with ``expert_major[r] =
    source_major[idx[r]]`` (expert ascending, source ascending within an
    expert — i.e. the global stable order restricted to this rank's experts).
    """
    n_src, n_e = recv_counts.shape
    starts = np.zeros((n_src, n_e), dtype=np.int64)
    flat = recv_counts.reshape(-1)
    starts.reshape(-1)[1:] = np.cumsum(flat)[:-1]
    out = []
    for e in range(n_e):
        for s in range(n_src):
            c = int(recv_counts[s, e])
            if c:
                out.append(np.arange(starts[s, e], starts[s, e] + c, dtype=np.int64))
    return np.concatenate(out) if out else np.zeros(0, dtype=np.int64)


class CudaOps:
    """Row compute on the GPU through the C-ABI (libmoe_b200.so)."""

    def __init__(self, config: ModelConfig, local_cfg: ModelConfig, router_weight, local_weights: ExpertWeights,
                 max_tokens: int, device):
        from .layer import MoELayer, _ptr, _stream_ptr, upload_weights  # noqa: F401

        self.device = device
        self.lib = _lib.load()
        # router: a full-E layer with placeholder expert stacks (routing only)
        E, d = config.num_experts, config.hidden_dim
        z = np.zeros((E * d, 8), np.float32)
        self.router = MoELayer(ModelConfig(E, config.top_k, d, 8, config.gating),
                               ExpertWeights(z, z, np.zeros((E * 8, d), np.float32)), router_weight,
                               max_tokens=max_tokens, device=device)
        self.w = upload_weights(local_weights, local_cfg, device)
        self.local_cfg = local_cfg
        self.cfg1 = _lib.config_struct(local_cfg.num_experts, 1, self.w.hidden_pad, self.w.ffn_pad,
                                       GATING_CODE[Gating(local_cfg.gating)])
        self.cfgk = _lib.config_struct(E, config.top_k, self.w.hidden_pad, self.w.ffn_pad, GATING_CODE[Gating(config.gating)])
        self._ws = None
        self._ws_bytes = 0
        self._ptr, self._stream = _ptr, _stream_ptr

    def route(self, x):
        r = self.router.route(x)
        return (r["indices"], r["weights"], r["counts"].clone(), r["forward"].clone(), r["inverse"].clone())

    def permute(self, x, fwd, k):
        xb = x.to(torch.bfloat16)
        if xb.shape[1] != self.w.hidden_pad:  # rows are gathered in 16-byte units at the padded width
            xb = torch.nn.functional.pad(xb, (0, self.w.hidden_pad - xb.shape[1]))
        xb = xb.contiguous()
        idx = (fwd // k).to(torch.int32).contiguous()
        return self.gather_rows(xb, idx)

    def gather_rows(self, src, idx):
        n = idx.numel()
        dst = torch.empty((n,) + tuple(src.shape[1:]), dtype=src.dtype, device=self.device)
        row_bytes = src[0].numel() * src.element_size() if src.shape[0] else 16
        _lib.check(self.lib.moe_b200_gather_rows(n, row_bytes, self._ptr(src), self._ptr(idx), self._ptr(dst),
                                                 self._stream(self.device)), "gather_rows")
        return dst

    def _down_splits(self, tokens):
        s = ctypes.c_int(0)
        _lib.check(self.lib.moe_b200_down_splits(ctypes.byref(self.cfgk), max(int(tokens), 1), ctypes.byref(s)),
                   "down_splits")
        return s.value

    def expert_ffn(self, counts, xp, global_tokens):
        """Local expert rows; the down projection uses the K-split count of the
        single-GPU forward over ``global_tokens`` tokens, so every row is
        bit-identical to that forward's."""
        n = xp.shape[0]
        out = torch.empty((n, self.w.hidden_pad), dtype=torch.float32, device=self.device)
        if n == 0:
            return out
        splits = self._down_splits(global_tokens)
        need = ctypes.c_size_t(0)
        # the split count falls as the batch grows: size for the largest (1 token)
        _lib.check(self.lib.moe_b200_expert_ffn_workspace_size(ctypes.byref(self.cfg1), n, self._down_splits(1),
                                                               ctypes.byref(need)), "ws")
        if need.value > self._ws_bytes:
            self._ws_bytes = int(need.value * 1.25)
            self._ws = torch.empty(self._ws_bytes, dtype=torch.uint8, device=self.device)
            _lib.check(self.lib.moe_b200_workspace_init(ctypes.byref(self.cfg1), n, self._ptr(self._ws),
                                                        self._ws_bytes, self._stream(self.device)), "ws_init")
        c = counts.to(torch.int32).contiguous()
        _lib.check(self.lib.moe_b200_expert_ffn(ctypes.byref(self.cfg1), n, splits, self._ptr(c), self._ptr(xp),
                                                self._ptr(self.w.gate), self._ptr(self.w.up), self._ptr(self.w.down),
                                                self._ptr(out), self._ptr(self._ws), self._ws_bytes,
                                                self._stream(self.device)), "expert_ffn")
        return out

    def _ensure_ws(self, n, splits_max):
        need = ctypes.c_size_t(0)
        _lib.check(self.lib.moe_b200_expert_ffn_workspace_size(ctypes.byref(self.cfg1), n, splits_max,
                                                               ctypes.byref(need)), "ws")
        if need.value > self._ws_bytes:
            self._ws_bytes = int(need.value * 1.25)
            self._ws = torch.empty(self._ws_bytes, dtype=torch.uint8, device=self.device)
            _lib.check(self.lib.moe_b200_workspace_init(ctypes.byref(self.cfg1), n, self._ptr(self._ws),
                                                        self._ws_bytes, self._stream(self.device)), "ws_init")

    def expert_ffn_return(self, counts, xp, global_tokens, peers, done, epoch):
        """Local expert FFN over the received rows with the peer-memory return
        fused into its K-split reduction (moe_b200_ep_p2p_ffn_return)."""
        n = xp.shape[0]
        splits = self._down_splits(global_tokens)
        if n:
            self._ensure_ws(n, self._down_splits(1))
        c = counts.to(torch.int32).contiguous()
        self._keep_ret = c
        _lib.check(self.lib.moe_b200_ep_p2p_ffn_return(
            ctypes.byref(self.cfg1), n, splits, self._ptr(c), self._ptr(xp), self._ptr(self.w.gate),
            self._ptr(self.w.up), self._ptr(self.w.down), peers, self._ptr(done), epoch,
            self._ptr(self._ws) if self._ws is not None else None, self._ws_bytes,
            self._stream(self.device)), "ep_p2p_ffn_return")

    def combine(self, rows, inv, w, B):
        y = torch.empty((B, rows.shape[1]), dtype=torch.float32, device=self.device)
        _lib.check(self.lib.moe_b200_combine_rows(ctypes.byref(self.cfgk), B, self._ptr(rows), self._ptr(inv),
                                                  self._ptr(w), self._ptr(y), _lib.DTYPE_F32,
                                                  self._stream(self.device)), "combine_rows")
        return y


class ExpertParallelMoE:
    """One MoE layer with experts sharded over the ranks of ``group``."""

    def __init__(self, config: ModelConfig, router_weight, weights_local: ExpertWeights, max_tokens: int,
                 group=None, device=None, ops=None, transport: str = "collective"):
        """``transport``: "collective" (torch.distributed all-to-alls) or "p2p"
        (rows written straight into the peers' buffers, PeerExchange)."""
        self.config = config
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.ranges = expert_ranges(config.num_experts, self.world)
        lo, hi = self.ranges[self.rank]
        self.local_cfg = ModelConfig(hi - lo, 1, config.hidden_dim, config.ffn_dim, config.gating)
        self.device = torch.device(device or "cuda")
        self.ops = ops or CudaOps(config, self.local_cfg, router_weight, weights_local, max_tokens, self.device)
        if transport not in ("collective", "p2p"):
            raise ValueError(f"transport must be 'collective' or 'p2p', got {transport!r}")
        self.p2p = PeerExchange(self, max_tokens) if transport == "p2p" else None

    def _a2a(self, out, inp, out_splits, in_splits):
        if self.world == 1:
            out.copy_(inp)
            return
        dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits, group=self.group)

    def forward(self, x: torch.Tensor, global_tokens: int | None = None) -> torch.Tensor:
        """This rank's token shard -> its output rows.  ``global_tokens``: see
        ``PeerExchange.forward`` (the collective transport learns it from the
        counts exchange)."""
        if self.p2p is not None:
            return self.p2p.forward(x, global_tokens)
        cfg = self.config
        k, E, d = cfg.top_k, cfg.num_experts, cfg.hidden_dim
        B = x.shape[0]
        idx, w, counts, fwd, inv = self.ops.route(x)
        xp = self.ops.permute(x, fwd, k)  # local expert-major rows (bf16)
        # counts exchange (the one host sync): per (src, local expert), plus each
        # source's token count (the global batch fixes the down K-split count)
        counts_h = counts.to("cpu", torch.int64).numpy() if counts.is_cuda else counts.numpy().astype(np.int64)
        send_counts = np.concatenate([np.append(counts_h[lo:hi], B) for lo, hi in self.ranges])
        send_t = torch.from_numpy(send_counts)
        n_loc = self.local_cfg.num_experts
        if self.world > 1:
            split = [hi - lo + 1 for lo, hi in self.ranges]
            recv_split = [n_loc + 1] * self.world
            dev = self.device if dist.get_backend(self.group) == "nccl" else torch.device("cpu")
            rc = torch.zeros(self.world * (n_loc + 1), dtype=torch.int64, device=dev)
            dist.all_to_all_single(rc, send_t.to(dev), output_split_sizes=recv_split, input_split_sizes=split,
                                   group=self.group)
            recv_all = rc.cpu().numpy().reshape(self.world, n_loc + 1)
        else:
            recv_all = send_counts.reshape(1, n_loc + 1)
        global_tokens = int(recv_all[:, -1].sum())
        recv_counts = recv_all[:, :-1]
        send_rows = [int(counts_h[lo:hi].sum()) for lo, hi in self.ranges]
        recv_rows = [int(r) for r in recv_counts.sum(axis=1)]
        # dispatch
        recv = torch.empty((sum(recv_rows), xp.shape[1]), dtype=xp.dtype, device=xp.device)
        self._a2a(recv, xp, recv_rows, send_rows)
        # source-major -> expert-major, local FFN, and back
        order = source_major_to_expert_major(recv_counts)
        order_t = torch.from_numpy(order.astype(np.int32)).to(xp.device)
        inv_order = np.empty_like(order)
        inv_order[order] = np.arange(order.size)
        inv_order_t = torch.from_numpy(inv_order.astype(np.int32)).to(xp.device)
        xe = self.ops.gather_rows(recv, order_t)
        local_counts = torch.from_numpy(recv_counts.sum(axis=0).astype(np.int32)).to(xp.device)
        ye = self.ops.expert_ffn(local_counts, xe, global_tokens)
        ys = self.ops.gather_rows(ye, inv_order_t)
        # combine: rows go home in the order they were sent
        back = torch.empty((sum(send_rows), ys.shape[1]), dtype=ys.dtype, device=ys.device)
        self._a2a(back, ys, send_rows, recv_rows)
        y = self.ops.combine(back, inv, w, B)
        return y[:, :d]


class PeerExchange:
    """The expert-parallel exchanges over peer memory (libmoe_b200 ``ep_p2p``).

    Each rank allocates its exchange buffers (counts, epoch flags, received
    rows and ids, returned outputs) with CUDA IPC handles; the handles are
    all-gathered over ``group`` once, and every rank maps every peer's
    buffers.  A forward then writes rows straight into the owners' buffers
    (dispatch fused with the local gather) and the expert outputs straight
    back into the home ranks' buffers, with device-side epoch flags instead
    of library all-to-alls.  Nothing synchronises with the host: the local
    expert FFN is laid out for the worst case and takes its per-expert counts
    from the all-gathered matrix on the device, so the forward is
    asynchronous, and with device-side epochs a captured CUDA graph of it
    replays correctly (after one eager forward has sized the workspace).
    """

    def __init__(self, ep: "ExpertParallelMoE", max_tokens: int):
        ops = ep.ops
        self.ep, self.ops, self.lib = ep, ops, ops.lib
        n, me = ep.world, ep.rank
        if n > _lib.EP_MAX_RANKS:
            raise ValueError(f"at most {_lib.EP_MAX_RANKS} ranks")
        E, k = ep.config.num_experts, ep.config.top_k
        d = ops.w.hidden_pad
        n_loc = ep.local_cfg.num_experts
        self.max_tokens = max_tokens
        # peers size their writes by their OWN batches: agree on every rank's
        # bound first, so the receive buffers cover the largest sender
        if n > 1:
            bounds = [None] * n
            dist.all_gather_object(bounds, int(max_tokens), group=ep.group)
        else:
            bounds = [int(max_tokens)]
        self.rank_max_tokens = [int(b) for b in bounds]
        # the layer's batch when every rank runs its bound (the default
        # global_tokens of forward: it fixes the down K-split count)
        self.global_tokens = sum(self.rank_max_tokens)
        # worst case: every token of every rank sends min(k, E_local) rows here
        self.r_max = max(1, sum(self.rank_max_tokens) * min(k, n_loc))
        t_max = max(1, max_tokens * k)
        sizes = {"counts": n * E * 4, "flags": 3 * n * 8, "rows": self.r_max * d * 2,
                 "ids": self.r_max * 8, "home": t_max * d * 4}
        self._own, handles = {}, {}
        for name, nbytes in sizes.items():
            p = ctypes.c_void_p()
            h = ctypes.create_string_buffer(64)
            _lib.check(self.lib.moe_b200_ipc_alloc(nbytes, ctypes.byref(p), h), "ipc_alloc")
            self._own[name] = p.value
            handles[name] = h.raw
        gathered = [None] * n
        if n > 1:
            dist.all_gather_object(gathered, handles, group=ep.group)
        else:
            gathered = [handles]
        self.peers = _lib.EpPeers()
        self._opened = []
        for r in range(n):
            for name in sizes:
                if r == me:
                    ptr = self._own[name]
                else:
                    p = ctypes.c_void_p()
                    _lib.check(self.lib.moe_b200_ipc_open(gathered[r][name], ctypes.byref(p)), "ipc_open")
                    ptr = p.value
                    self._opened.append(ptr)
                getattr(self.peers, name)[r] = ptr
        for r, (lo, _) in enumerate(ep.ranges):
            self.peers.expert_lo[r] = lo
        self.peers.expert_lo[n] = E
        self.peers.n, self.peers.me = n, me
        dev = ep.device
        # device-side epochs {counter, current}: every call passes epoch 0, the
        # counts kernel advances it, so a captured CUDA graph replays correctly
        self.epoch_dev = torch.zeros(2, dtype=torch.int64, device=dev)
        self.peers.epoch_dev = self.epoch_dev.data_ptr()
        self.done = torch.zeros(2, dtype=torch.int32, device=dev)  # dispatch / return CTA counters
        self.inv_identity = torch.arange(t_max, dtype=torch.int32, device=dev)
        # local views of the own buffers
        self.counts_local = _device_view(self._own["counts"], (n, E), torch.int32, dev)
        self.rows_local = _device_view(self._own["rows"], (self.r_max, d), torch.bfloat16, dev)
        self.home_local = _device_view(self._own["home"], (t_max, d), torch.float32, dev)
        if n > 1:
            dist.barrier(group=ep.group)  # every rank mapped every buffer

    def forward(self, x: torch.Tensor, global_tokens: int | None = None) -> torch.Tensor:
        """Asynchronous (no host synchronisation).
        ``global_tokens`` is the layer's total batch over all ranks; it fixes
        the down K-split count so every row matches the single-GPU forward bit
        for bit.  Default: the sum of the ranks' ``max_tokens`` (all-gathered
        at construction), i.e. every rank running a full batch; a rank whose
        batch is partial passes the true total (there is no host
        synchronisation here to learn it)."""
        ep, ops, lib = self.ep, self.ops, self.lib
        cfg = ep.config
        k, d = cfg.top_k, cfg.hidden_dim
        B = x.shape[0]
        if global_tokens is None:
            global_tokens = self.global_tokens if ep.world > 1 else B
        if B > self.max_tokens:
            raise ValueError(f"{B} tokens > max_tokens {self.max_tokens}")
        s = ops._stream(ep.device)
        peers = ctypes.byref(self.peers)
        e = 0  # device-side epoch
        r = ops.router.route(x)
        xb = x.to(torch.bfloat16)
        if xb.shape[1] != ops.w.hidden_pad:
            xb = torch.nn.functional.pad(xb, (0, ops.w.hidden_pad - xb.shape[1]))
        xb = xb.contiguous()
        self._keep = (xb, r)  # alive while the launches run
        _lib.check(lib.moe_b200_ep_p2p_counts(ctypes.byref(ops.cfgk), B * k, ops._ptr(r["indices"]), peers, e, s),
                   "ep_p2p_counts")
        # dispatch waits for every source's counts (flag set 0) on the device
        _lib.check(lib.moe_b200_ep_p2p_dispatch(ctypes.byref(ops.cfgk), B, ops._ptr(xb), ops._ptr(r["indices"]),
                                                ops._ptr(r["forward"]), ops._ptr(r["offsets"]), peers,
                                                ops._ptr(self.done[0:1]), e, s), "ep_p2p_dispatch")
        # local expert FFN over the received rows (flag set 1 awaited on the
        # device, counts from the all-gathered matrix), the return to the home
        # ranks fused into its K-split reduction
        splits = ops._down_splits(global_tokens)
        ops._ensure_ws(self.r_max, max(splits, ops._down_splits(1)))
        _lib.check(lib.moe_b200_ep_p2p_ffn_return_async(
            ctypes.byref(ops.cfg1), self.r_max, splits, ops._ptr(self.rows_local), ops._ptr(ops.w.gate),
            ops._ptr(ops.w.up), ops._ptr(ops.w.down), peers, ops._ptr(self.done[1:2]), e, ops._ptr(ops._ws),
            ops._ws_bytes, s), "ep_p2p_ffn_return_async")
        _lib.check(lib.moe_b200_ep_p2p_wait(peers, 2, e, s), "ep_p2p_wait")
        y = ops.combine(self.home_local[: B * k], self.inv_identity[: B * k], r["weights"], B)
        return y[:, :d]

    def close(self):
        torch.cuda.synchronize(self.ep.device)
        for p in self._opened:
            self.lib.moe_b200_ipc_close(ctypes.c_void_p(p))
        self._opened = []
        for p in self._own.values():
            self.lib.moe_b200_ipc_free(ctypes.c_void_p(p))
        self._own = {}


def _device_view(ptr: int, shape, dtype, device) -> torch.Tensor:
    """A torch tensor over library-owned device memory (no copy, not owned)."""
    n = int(np.prod(shape))
    nbytes = n * torch.empty((), dtype=dtype).element_size()
    # wrap the pointer through __cuda_array_interface__ (torch does not own it)
    class _Arr:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}
    t = torch.as_tensor(_Arr(), device=device)
    return t.view(dtype).view(*shape)
