"""CPU shard backend for the distributed tests: the PHASE_UP / PHASE_DOWN
contract of ``CudaShardBackend`` (vfmm_evaluate_shard, include/vfmm.h)
computed by the numpy oracle.  Test infrastructure only: it lets the gloo
tests check the host orchestration and the decomposition arithmetic of
``paper_0809_1810_b200.distributed`` without a GPU."""
import numpy as np
import torch

from oracle import fmm_oracle as O


def _il_count(occ_k, k):
    """Per destination cell of level k: number of non-empty interaction-list sources."""
    m = 2**k
    iy, ix = np.divmod(np.arange(m * m), m)
    cnt = np.zeros(m * m, dtype=np.int64)
    for dy in range(-3, 4):
        for dx in range(-3, 4):
            if max(abs(dx), abs(dy)) < 2:
                continue
            okx = np.where(ix % 2 == 0, (dx >= -2) & (dx <= 3), (dx >= -3) & (dx <= 2))
            oky = np.where(iy % 2 == 0, (dy >= -2) & (dy <= 3), (dy >= -3) & (dy <= 2))
            sx, sy = ix + dx, iy + dy
            sel = okx & oky & (sx >= 0) & (sx < m) & (sy >= 0) & (sy < m)
            src = np.where(sel, sy * m + sx, 0)
            cnt += sel & (occ_k[src] > 0)
    return cnt


class OracleShardBackend:
    def up(self, shard, config, domain):
        c = shard.cols.numpy()
        x, y, g, s = c[0], c[1], c[2], c[3]
        lv, p = config.levels, config.order
        self.dom = (domain.xmin, domain.ymin, domain.side)
        self.n = c.shape[1]
        keys = O.leaf_keys(x, y, lv, *self.dom) if self.n else np.zeros(0, np.int64)
        self.tree = O.Tree(keys, lv, *self.dom)
        lo, hi = shard.rows
        row = keys >> lv
        owned = (row >= lo) & (row < hi)
        t = self.tree
        self.z = (x + 1j * y)[t.order]
        self.xs, self.ys, self.gs, self.ss = x[t.order], y[t.order], g[t.order], s[t.order]
        mult = O.p2m_m2m(t, self.z, self.gs * owned[t.order], p)
        occ = O.Tree(keys[owned], lv, *self.dom).counts
        self.mult_flat = torch.from_numpy(
            np.concatenate([mult[k].ravel() for k in range(2, lv + 1)]).view(np.float64).copy())
        self.occ_flat = torch.from_numpy(
            np.concatenate([occ[k] for k in range(lv + 1)]).astype(np.int32))
        return self.mult_flat, self.occ_flat

    def down(self, shard, config, domain, counters=True):
        lv, p = config.levels, config.order
        t = self.tree
        lo, hi = shard.rows
        flat = self.mult_flat.numpy().view(np.complex128)
        mult, off = {}, 0
        for k in range(2, lv + 1):
            mult[k] = flat[off: off + 4**k * (p + 1)].reshape(4**k, p + 1)
            off += 4**k * (p + 1)
        occ, off = {}, 0
        for k in range(lv + 1):
            occ[k] = self.occ_flat.numpy()[off: off + 4**k].astype(np.int64)
            off += 4**k
        local_counts = t.counts
        t.counts = occ  # global occupancy for the interaction-list emptiness test
        loc, _ = O.m2l(t, mult, p)
        O.l2l(t, loc, p)
        t.counts = local_counts
        m2l = 0
        for k in range(2, lv + 1):
            first_row = (np.arange(2**k) << (lv - k))
            own_rows = (first_row >= lo) & (first_row < hi)
            per = _il_count(occ[k], k).reshape(2**k, 2**k)
            m2l += int(per[own_rows].sum())
        gauss = getattr(config.kernel, "value", config.kernel) == "gaussian_blob"
        far = O.to_velocity(O.l2p(t, loc, self.z)) if self.n else np.zeros((0, 2))
        near, _ = O.p2p(t, self.xs, self.ys, self.gs, self.ss, gauss)
        near_pairs = 0
        m = 2**lv
        for leaf in np.flatnonzero(t.counts[lv]):
            if lo <= leaf // m < hi:
                nb = sum(b - a for a, b in O.neighbourhood(t, leaf))
                near_pairs += int(t.leaf_starts[leaf + 1] - t.leaf_starts[leaf]) * int(nb - 1)
        vel_sorted = far + near
        vel = np.zeros((self.n, 2))
        vel[t.order] = vel_sorted
        return torch.from_numpy(vel.T.copy()), m2l, near_pairs
