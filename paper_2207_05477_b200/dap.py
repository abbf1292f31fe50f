"""Dynamic Axial Parallelism (DAP) on the sm_100a engine.

The reference's sharded model (``DapPar``, src/harness.py:262-293, and the
``par.*`` call sites of src/model.py:312-398) split over ``d`` workers:

* MSA [S, R, c_m] by sequence: worker k holds sequences k*s .. k*s+s-1
  (s = S/d) as a token-major [s*R, c_m] buffer;
* pair [R, R, c_z] by row: worker k holds rows k*r .. k*r+r-1 (r = R/d).

Per block (the reference's "mini" table, src/planner.py:46-50):

* MSA row attention: pair bias from the local pair rows, all-gathered into
  the full [H, R, R] bias; backward reduce-scatters its gradient;
* MSA column attention: all-to-all into a residue-column shard [S, r, c_m],
  attention (+ gated output projection + residual) there, all-to-all back;
  backward the same pair of all-to-alls on the gradient;
* outer product mean: this worker's sequences give a partial [R*k, R*k]
  sum, reduce-scattered (fp32) into the local rows; backward all-gathers
  d(num);
* triangle attention start: as MSA row attention, on the pair rows;
* triangle attention end: all-to-all into the column shard [R, r, c_z], whose
  tokens the attention reads through the same (batch, position) strides as
  the unsharded triangle-end variant; all-to-all back;
* transitions, LayerNorms, embeddings and the loss are row-local; the loss
  and every parameter gradient are partial sums, closed by one all-reduce of
  the pooled grad region (``dap_step``).

Each collective exchanges contiguous dim-0 chunks (NCCL all_to_all_single,
all_gather_into_tensor, reduce_scatter_tensor); the ``evo_swap01`` kernel is
the re-layout on either side (e.g. [s, R, C] = [s, d, r*C] -> [d, s, r*C]).
The reference transposes around its collectives as well (src/model.py:335-340).
"""

from __future__ import annotations

import numpy as np

from . import ops
from .engine import F32, BlockEngine, DeviceFeatures, Variant
from .errors import ContractError
from .parallel import Comm, GridConfig

MODULE = {"row_attn": "msa_row_attn", "col_attn": "msa_col_attn", "tri_start": "tri_start",
          "tri_end": "tri_end"}


class DapEngine(BlockEngine):
    """One DAP worker's block engine: ``BlockEngine`` on the shard, with the
    collectives in its sharding hooks and around the column-wise modules."""

    def __init__(self, cfg, store, act_dtype, comm: Comm, arena_mb: int = 96):
        d, k = comm.size, comm.rank
        S, R = cfg.n_seq, cfg.n_res
        if S % d or R % d:
            raise ContractError(f"plan.dap: cannot shard n_seq={S} / n_res={R} over {d} workers")
        if cfg.trimul:
            raise ContractError("plan.dap: TriangleMultiplication is not sharded (mini block only)")
        super().__init__(cfg, store, act_dtype, arena_mb=arena_mb)
        self.comm, self.d, self.k = comm, d, k
        s, r = S // d, R // d
        self.s_loc = s
        self.s0, self.r0, self.r_loc = k * s, k * r, r
        self.opm_num_dtype = F32          # partial sums travel in fp32
        self.branch_streams = False       # collectives stay on the current stream
        # local geometries (engine.variants for the unsharded ones)
        self.var = {
            "row_attn": Variant("row_attn", s, R, R, 1, R, 1, "msa", True, False,
                                moff=k * s * R, ni=r, nj=R),
            "col_attn": Variant("col_attn", r, S, 1, r, 1, R, "msa", False, False, moff=k * r),
            "tri_start": Variant("tri_start", r, R, R, 1, R, 1, "pair", True, False,
                                 moff=k * r * R, ni=r, nj=R),
            "tri_end": Variant("tri_end", r, R, 1, r, 1, R, "pair", True, True,
                               moff=k * r, ni=R, nj=r),
        }

    # -- sharding hooks ---------------------------------------------------------------

    def _gather_bias(self, nb, v: Variant):
        """[H, r, R] local rows -> [H, R, R] (src/model.py:317)."""
        H = nb.shape[0]
        g = self.comm.allgather(nb, MODULE[v.name])                   # [d*H, r, R] rank-major
        return ops.swap01(g, self.d, H).view(H, self.cfg.n_res, self.cfg.n_res)

    def _scatter_dbias(self, dnb, v: Variant):
        """[H, R, R] partial over this worker's batches -> its rows, summed."""
        H = dnb.shape[0]
        t = ops.swap01(dnb, H, self.d)                                # [d, H, r, R]
        return self.comm.reducescatter_sum(t.view(self.d * H, -1), MODULE[v.name])

    def _opm_reduce(self, num):
        return self.comm.reducescatter_sum(num, "opm")                # [r*k, R*k] rows

    def _opm_gather(self, dnum):
        return self.comm.allgather(dnum, "opm")

    def _feat_rows(self, feats: DeviceFeatures):
        R = self.cfg.n_res
        ms = slice(self.s0 * R, (self.s0 + self.s_loc) * R)
        ps = slice(self.r0 * R, (self.r0 + self.r_loc) * R)
        return feats.msa_feat[ms], feats.pair_feat[ps], feats.msa_mask[ms]

    # -- row shard <-> column shard ---------------------------------------------------

    def _to_cols(self, x, n, module):
        """[n*R, C] (rows n, all R columns) -> [d*n*r, C] (all d*n rows, r columns)."""
        t = ops.swap01(x, n, self.d)                                  # [d, n, r, C]
        return self.comm.alltoall(t, module)

    def _to_rows(self, t, n, module, out=None):
        """Inverse of ``_to_cols``."""
        u = self.comm.alltoall(t, module)                            # [d(src), n, r, C]
        return ops.swap01(u, self.d, n, out=out)                      # [n, d, r, C]

    # -- branches ------------------------------------------------------------------------

    def msa_branch_fwd(self, i, msa_in, pair_in, feats):
        p = f"block{i}"
        msa, s1 = self.attn_fwd(msa_in, f"{p}.row_attn", self.var["row_attn"], feats, pair=pair_in)
        t, s2 = self.attn_fwd(self._to_cols(msa, self.s_loc, "msa_col_attn"), f"{p}.col_attn",
                              self.var["col_attn"], feats)
        msa = self._to_rows(t, self.s_loc, "msa_col_attn")
        del t
        msa, s3 = self.trans_fwd(msa, f"{p}.msa_trans")
        return msa, (s1, s2, s3)

    def msa_branch_bwd(self, i, d_msa, d_pair_acc, saved, feats, late=None, d_act=None):
        p = f"block{i}"
        s1, s2, s3 = saved
        self.trans_bwd(d_msa, s3, f"{p}.msa_trans", d_act=d_act)
        dt_ = self._to_cols(d_msa, self.s_loc, "msa_col_attn")
        self.attn_bwd(dt_, s2, f"{p}.col_attn", self.var["col_attn"], feats)
        self._to_rows(dt_, self.s_loc, "msa_col_attn", out=d_msa)
        del dt_
        self.attn_bwd(d_msa, s1, f"{p}.row_attn", self.var["row_attn"], feats, dpair=d_pair_acc)

    def pair_branch_fwd(self, i, pair_mid, feats):
        p = f"block{i}"
        pair, s1 = self.attn_fwd(pair_mid, f"{p}.tri_start", self.var["tri_start"], feats)
        t, s2 = self.attn_fwd(self._to_cols(pair, self.r_loc, "tri_end"), f"{p}.tri_end",
                              self.var["tri_end"], feats)
        pair = self._to_rows(t, self.r_loc, "tri_end")
        del t
        pair, s3 = self.trans_fwd(pair, f"{p}.pair_trans")
        return pair, ([], s1, s2, s3)

    def pair_branch_bwd(self, i, d_pair, saved, feats, opm_nxt=False, d_act=None):
        p = f"block{i}"
        _, s1, s2, s3 = saved
        self.trans_bwd(d_pair, s3, f"{p}.pair_trans", d_act=d_act)
        dt_ = self._to_cols(d_pair, self.r_loc, "tri_end")
        self.attn_bwd(dt_, s2, f"{p}.tri_end", self.var["tri_end"], feats)
        self._to_rows(dt_, self.r_loc, "tri_end", out=d_pair)
        del dt_
        self.attn_bwd(d_pair, s1, f"{p}.tri_start", self.var["tri_start"], feats)

    def forward_backward(self, feats, n_cycles: int = 1, recompute: bool = False, grad_ready=None):
        self.comm.phase = "fwd"
        out = super().forward_backward(feats, n_cycles, recompute=recompute, grad_ready=grad_ready)
        self.comm.phase = "bwd"
        return out

    def loss(self, msa, pair):
        self.comm.phase = "bwd"          # everything after the forward is backward traffic
        return super().loss(msa, pair)

    def gather_outputs(self, msa, pair):
        """Full (msa, pair) for verification (module "output", not on the step)."""
        return self.comm.allgather(msa, "output"), self.comm.allgather(pair, "output")


def dap_step(engine: DapEngine, feats, world: Comm, grid: GridConfig, n_cycles: int = 1,
             step: int = 0, recompute: bool = False):
    """``_dap_step`` (src/harness.py:355-389): sharded fwd+bwd, then ONE
    all-reduce of the pooled grad region over the world (the DAP partial sums
    and, with dp > 1, the replica average) and of the loss."""
    engine.comm.step = world.step = step
    loss, outs = engine.forward_backward(feats, n_cycles, recompute=recompute)
    world.phase = "grad-sync"
    g = engine.grad_region()
    world.allreduce_sum(g, "grad_sync")
    lt = loss.reshape(1).clone()
    world.allreduce_sum(lt, "loss")
    if grid.dp > 1:
        g.mul_(np.float32(1.0 / grid.dp).item())
        lt.mul_(np.float32(1.0 / grid.dp).item())
    return lt, outs
