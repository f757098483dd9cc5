"""K-sharded MPPI step across GPUs ("the sampling for loop ...
is run completely in parallel", :320 the sums over k).

Rank r of G owns global samples [r K/G, (r+1) K/G).  Noise counters use the global k, so the
shards' noise is disjoint and its union is the single-GPU noise bit for bit.  The only
cross-rank data are two tiny collectives on the step's stream (NCCL over NVLink via
torch.distributed):
  1. allreduce MIN of the int64 (cost, k) key  -> S_min and k* (8 bytes)
  2. allreduce SUM of [eta, A[T][m]]           -> normaliser and weighted noise sum ((1+Tm)*4 B)
after which every rank applies the same update, keeping U a bit-identical replica.
"""
import torch
import torch.distributed as dist


def shard_range(K, rank, world):
    """(k_offset, K_loc) of `rank`; K must divide evenly and K_loc must be a multiple of 4."""
    if K % world:
        raise ValueError("K=%d is not divisible by world=%d" % (K, world))
    K_loc = K // world
    if K_loc % 4:
        raise ValueError("K/world=%d must be a multiple of 4" % K_loc)
    return rank * K_loc, K_loc


class ShardedMPPI:
    """Runs one MPPI step of `stepper` (an MPPI context created with rank/world) with the
    cross-rank reductions.  `stepper` needs rollout_costs / accumulate / apply with the
    semantics of the split-phase C ABI (include/mppi.h); combine="gather" uses the one-collective
    form instead (accumulate_record / apply_gathered: every rank's [key, eta, A] record against its
    own minimum, one all-gather, the rescale in rank order -- MPPI_OPTION_GATHER_COMBINE)."""

    def __init__(self, stepper, group=None, combine="allreduce"):
        if combine not in ("allreduce", "gather"):
            raise ValueError("combine must be 'allreduce' or 'gather'")
        self.stepper = stepper
        self.group = group
        self.combine = combine
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1

    def optimize(self, x0, U, seed=0, step=0, noise=None):
        s = self.stepper
        _, key = s.rollout_costs(x0, U, seed, step, noise)
        if self.combine == "gather":
            rec = s.accumulate_record()
            if self.world > 1:
                recs = [torch.empty_like(rec) for _ in range(self.world)]
                dist.all_gather(recs, rec, group=self.group)
                rec = torch.stack(recs)
            else:
                rec = rec.unsqueeze(0)
            s.apply_gathered(U, rec)
            return U
        if self.world > 1:
            dist.all_reduce(key, op=dist.ReduceOp.MIN, group=self.group)
        buf = s.accumulate(key)
        if self.world > 1:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)
        s.apply(U, buf)
        return U
