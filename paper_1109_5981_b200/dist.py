"""Multi-GPU plumbing for the LSRN C ABI (argument marshalling only).

The paper's MPI design (§4.3): each process holds a block of rows of
A (tall) or columns (wide, Alg. 2), forms its partial sketch G_p A_p, the
partials are reduced, and every iteration needs one reduction of a short
vector.  Here each rank is one GPU; the reductions are NCCL allreduces issued
*inside* liblsrn.so on the library's stream (the iteration loop is one CUDA
graph that contains them).  This module only

  * splits the long dimension into contiguous shards (`shard_bounds`), so that
    rank p owns long indices [lo, hi) and passes (lo, cnt) to the C ABI, which
    uses the GLOBAL index j = lo + local in the Philox counter (C9):
    the sum of the partial sketches is independent of the rank count;
  * moves rank 0's NCCL unique id to every rank through torch.distributed
    (`exchange_unique_id`), which the library turns into its communicator;
  * or, without NCCL (`host_context`), hands the library host-staged
    collectives over any torch.distributed backend (gloo, MPI): the library
    copies the operand to the host and calls back for the sum / broadcast --
    the paper's own MPI_Reduce / MPI_Bcast / MPI_Allreduce.

Nothing here computes any part of the method.
"""
import torch.distributed as dist


def shard_bounds(L, world, rank):
    """Contiguous shard [lo, hi) of the long dimension L for `rank` of `world`.

    Shards differ in size by at most one row, cover [0, L) exactly once, and are
    ordered by rank (rank 0 starts at 0 and therefore owns the Tikhonov block,
    lsrn.h "Tikhonov").
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    if L < 0:
        raise ValueError("L must be >= 0")
    return (L * rank) // world, (L * (rank + 1)) // world


def exchange_unique_id(make_id, group=None):
    """Rank 0 calls make_id() (liblsrn's lsrn_nccl_unique_id); all ranks get its bytes."""
    if not dist.is_initialized():
        return make_id()
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def context(stream=None, group=None):
    """An lsrn.Context over all ranks of the default process group (NCCL id exchanged)."""
    from . import lsrn
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return lsrn.Context(stream=stream)
    nid = exchange_unique_id(lsrn.nccl_unique_id, group)
    return lsrn.Context(stream=stream, nranks=dist.get_world_size(group), rank=dist.get_rank(group), nccl_id=nid)


def host_context(stream=None, group=None):
    """An lsrn.Context over the ranks of `group` whose collectives are host-staged
    through torch.distributed (lsrn_ctx_set_host_collectives): no NCCL communicator,
    the iteration loop runs eagerly.  Works with the gloo backend (and on one GPU
    shared by several processes, since no kernel waits on another rank's kernel)."""
    import torch
    from . import lsrn
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    ctx = lsrn.Context(stream=stream, nranks=world, rank=rank)

    def allreduce(arr):
        t = torch.from_numpy(arr)          # shares the library's host buffer
        dist.all_reduce(t, group=group)

    def bcast(arr, root):
        t = torch.from_numpy(arr)
        dist.broadcast(t, src=dist.get_global_rank(group, root) if group is not None else root, group=group)
    ctx.set_host_collectives(allreduce, bcast)
    return ctx
