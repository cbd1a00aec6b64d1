"""Multi-GPU plumbing for the column-sharded greedy.

One process per GPU; torch.distributed supplies the process group (NCCL on GPUs, gloo in
the CPU tests) and is used only for setup: the column partition, the broadcast of the
NCCL unique id that the library's own communicator is built from, and max-over-ranks
timing, and (PEER mode) the one-time all-gather of every rank's CUDA-IPC handles.  The
per-iteration exchange happens inside librbg.so on the library's stream: PEER = P2P stores
of the maxloc records from the sweep kernel and NVLink reads of the pivot column by IMGS;
NCCL = one ncclAllGather of a {maxloc record, candidate column} slot per rank.

The paper distributes columns over "pivot cores" ("distributing N/P
columns" read as M/P, reading R11); here contiguous blocks, the last ranks taking the
remainder one column at a time.
"""
from __future__ import annotations


def partition(M_global: int, world: int, rank: int) -> tuple[int, int]:
    """(col_offset, M_loc) of `rank`: contiguous blocks, sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world or M_global < world:
        raise ValueError(f"cannot split {M_global} columns over {world} ranks")
    base, extra = divmod(M_global, world)
    offset = rank * base + max(0, rank - (world - extra))
    size = base + (1 if rank >= world - extra else 0)
    return offset, size


def broadcast_bytes(payload: bytes | None, group=None, src: int = 0) -> bytes:
    """Rank `src` sends `payload` (e.g. the 128-byte NCCL unique id) to every rank."""
    import torch.distributed as dist
    obj = [payload]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def nccl_unique_id(group=None) -> bytes:
    """rbg_get_unique_id on rank 0, broadcast over the process group."""
    import torch.distributed as dist
    from . import rbg
    uid = rbg.unique_id() if dist.get_rank(group) == 0 else None
    return broadcast_bytes(uid, group)


def max_over_ranks(x: float, group=None, device=None) -> float:
    """Multi-GPU timings are reported as the max over ranks (bench contract)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(x)
    if dist.get_backend(group) == "gloo":
        device = "cpu"                               # gloo reduces host tensors
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def all_gather_bytes(payload: bytes, group=None) -> list[bytes]:
    """Every rank's `payload` (e.g. its PEER CUDA-IPC handles), in rank order."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, payload, group=group)
    return out


def connect_peers(ctx, group=None):
    """PEER exchange setup: all-gather every rank's IPC handles and map them.  Every rank
    takes part in the all-gather even if its export failed (then every rank raises), so a
    failure never leaves the ranks in different collectives."""
    from . import rbg
    try:
        mine = ctx.peer_export()
    except rbg.RbgError:
        mine = None
    handles = all_gather_bytes(mine, group)
    if any(h is None for h in handles):
        raise rbg.RbgError(rbg.ESTATE, "a rank could not export its PEER handles")
    ctx.peer_connect(handles)
    return ctx


def sharded_context(S_local, w, tol: float, k_max: int, M_global: int, group=None, comm: str = "peer", **kw):
    """rbg.Context for this rank's column block of a `group`-wide sharded greedy.  comm="peer":
    records and the pivot column move over NVLink inside the kernels (CUDA IPC); "nccl": one
    ncclAllGather per iteration on a communicator shared by the ranks.  S_local must be this
    rank's partition(M_global, world, rank) block."""
    import torch.distributed as dist
    from . import rbg
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    off, m_loc = partition(M_global, world, rank)
    if S_local.shape[0] != m_loc:
        raise ValueError(f"rank {rank} holds {S_local.shape[0]} columns, partition says {m_loc}")
    if world == 1:
        return rbg.Context(S_local, w, tol, k_max, **kw)
    if comm == "peer":
        ctx = rbg.Context(S_local, w, tol, k_max, comm=rbg.COMM_PEER, rank=rank, world=world,
                          col_offset=off, M_global=M_global, **kw)
        return connect_peers(ctx, group)
    if comm != "nccl":
        raise ValueError(f"comm must be 'peer' or 'nccl', not {comm!r}")
    uid = nccl_unique_id(group)
    return rbg.Context(S_local, w, tol, k_max, comm=rbg.COMM_NCCL, rank=rank, world=world,
                       col_offset=off, M_global=M_global, nccl_id=uid, **kw)


class _DevPtr:
    """A device byte range as a torch tensor (zero copy, __cuda_array_interface__)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


def exchange_slots(ctx, group=None, stream=None):
    """The a4 exchange of an EXTERNAL context driven over the process group: every rank's
    {maxloc record, candidate column} send slot all-gathered into every rank's receive slots
    (rank p's bytes at recv + p * bytes), then rbg_iter_finish decides on the same records
    everywhere.  NCCL groups gather the device slots directly; gloo groups (CPU tests, several
    ranks sharing one GPU) stage them through host memory.  Call between iter_local and
    iter_finish; `stream` = the context's stream (the slot is read after it)."""
    import torch
    import torch.distributed as dist
    send, recv, nbytes = ctx.xchg_buffers()
    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    s_t = torch.as_tensor(_DevPtr(send, nbytes), device=dev)
    r_t = torch.as_tensor(_DevPtr(recv, nbytes * world), device=dev)
    if stream is not None:
        stream.synchronize()
    else:
        ctx.sync()
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(r_t, s_t, group=group)
        torch.cuda.current_stream(dev).synchronize()
        return
    h = s_t.cpu()
    parts = [torch.empty_like(h) for _ in range(world)]
    dist.all_gather(parts, h, group=group)
    r_t.copy_(torch.cat(parts))
    torch.cuda.current_stream(dev).synchronize()


def fold_over_ranks(fold, k: int, group=None):
    """Rank-order fold of a k x k complex matrix: rank p receives the running value from rank
    p - 1 (zeros on rank 0), applies `fold` (G -> G'), passes it to rank p + 1; the last rank's
    result is broadcast.  Returns it (numpy, G[i, j]) on every rank."""
    import numpy as np
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    buf = torch.zeros((k, k), dtype=torch.complex128, device=dev)
    ranks = dist.get_process_group_ranks(group) if group is not None else list(range(world))
    if rank > 0:
        dist.recv(buf, src=ranks[rank - 1], group=group)
    G = fold(buf.cpu().numpy())                      # buf[i, j] = G(i, j)
    buf.copy_(torch.from_numpy(np.ascontiguousarray(G)))
    if rank < world - 1:
        dist.send(buf, dst=ranks[rank + 1], group=group)
    dist.broadcast(buf, src=ranks[world - 1], group=group)
    return buf.cpu().numpy()


def sharded_reconstruct(ctx, tau2: float = 0.0, kr_max: int = 0, group=None):
    """Algorithm 4 on a column-sharded context: the Gram matrix R R^H is
    folded rank by rank in rank order (rbg_gram_fold: rank p adds its chunk partials onto the
    sum of ranks < p), the last rank's sum is broadcast, and every rank runs the eigen-step
    and X = Q V on the same G (rbg_reconstruct_gram), so sigma and X are replicated.  Equal to
    the single-GPU rbg_reconstruct bit for bit when every col_offset is a multiple of 4096
    (R33).  Returns (sigma, kr, X)."""
    G = fold_over_ranks(ctx.gram_fold, ctx.info()[0], group)
    return ctx.reconstruct_gram(G, tau2, kr_max)


def enrich_plan(counts: list[int], rank: int, M_global: int) -> tuple[int, int]:
    """(first_gid, M_global_new) of `rank` for one sharded enrichment round: the ranks'
    appended blocks are numbered in rank order after the current M_global columns, so the
    global column order is that of one context enriched with the concatenated blocks."""
    return M_global + sum(counts[:rank]), M_global + sum(counts)


def sharded_enrich(ctx, V_local, tol: float, rounds: int = 3, group=None, M_global: int | None = None):
    """Iterative refinement (reading R32) on a column-sharded context: each
    rank validates its own block of the validation set, appends its failing columns (not
    appended before) with global ids from enrich_plan, and the greedy continues on every rank.
    V_local is this rank's block of a validation set partitioned in rank order; M_global is the
    current total (default: the M_global the context was created with, tracked here).
    Returns (per-round max validation error over all ranks, passed)."""
    import numpy as np
    import torch.distributed as dist
    from . import rbg
    if hasattr(V_local, "is_cuda") and V_local.is_cuda:
        Vh = V_local                                   # validated in place, gathered on the device
    else:
        Vh = V_local.cpu().numpy() if hasattr(V_local, "cpu") else np.asarray(V_local)
    added = np.zeros(Vh.shape[0], bool)
    history = []
    total = M_global if M_global is not None else ctx.M_global

    def max_err(err):
        return max(all_gather_bytes(float(err.max()) if err.size else 0.0, group))

    for _ in range(rounds):
        err = ctx.validate(Vh)
        history.append(max_err(err))
        fail = (err >= tol) & ~added
        counts = all_gather_bytes(int(fail.sum()), group)
        if sum(counts) == 0:
            passed = all(all_gather_bytes(bool(np.all(err < tol)), group))
            return history, passed
        first, total_new = enrich_plan(counts, dist.get_rank(group), total)
        ctx.add_columns(rbg._rows(Vh, fail), first_gid=first, M_global=total_new)
        total = total_new
        added |= fail
        ctx.run()
    err = ctx.validate(Vh)
    history.append(max_err(err))
    return history, all(all_gather_bytes(bool(np.all(err < tol)), group))
