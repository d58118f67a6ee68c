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


def _touch(rows_k, lo, hi, sft):
    """Cell rows of a level whose leaf-row span intersects [lo, hi)."""
    return ((rows_k << sft) < hi) & (((rows_k + 1) << sft) > lo)


class OracleShardBackend:
    """PHASE_UP (strip-local partial multipoles), pack / unpack of the multipole
    exchange and PHASE_DOWN, in numpy.  Its exchange buffers use their own byte
    format (all ranks run the same backend): coarse = levels 2..kc of the
    multipoles masked to the cells touching the strip, then the occupancy of
    levels 0..kc; halo = two cell rows of every fine level, multipoles then
    occupancy."""

    def up(self, shard, config, domain):
        c = shard.cols.numpy()
        x, y, g, s = c[0], c[1], c[2], c[3]
        lv, p = config.levels, config.order
        self.lv, self.p, self.rows = lv, p, shard.rows
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
        # only owned particles carry circulation: fine cells of the strip are
        # complete, coarse cells straddling strips partial (linear in Gamma)
        self.mult = O.p2m_m2m(t, self.z, self.gs * owned[t.order], p)
        self.occ = {k: v.astype(np.int64) for k, v in O.Tree(keys[owned], lv, *self.dom).counts.items()}

    # ---- exchange ----
    def _coarse(self, kc):
        if kc < 2:
            return None
        lo, hi = self.rows
        parts = []
        for k in range(2, kc + 1):
            mk = 2**k
            m = self.mult[k].reshape(mk, mk, self.p + 1).copy()
            m[~_touch(np.arange(mk), lo, hi, self.lv - k)] = 0
            parts.append(m.ravel().view(np.float64))
        occ = np.concatenate([self.occ[k] for k in range(kc + 1)]).astype(np.float64)
        return torch.from_numpy(np.concatenate(parts + [occ]).view(np.uint8).copy())

    def _rows(self, kc, which):
        lo, hi = self.rows
        parts, occ = [], []
        for k in range(max(2, kc + 1), self.lv + 1):
            mk, sft = 2**k, self.lv - k
            r0 = (lo >> sft) if which == "down" else (hi >> sft) - 2
            parts.append(self.mult[k].reshape(mk, mk, self.p + 1)[r0: r0 + 2].ravel().view(np.float64))
            occ.append(self.occ[k].reshape(mk, mk)[r0: r0 + 2].ravel().astype(np.float64))
        return torch.from_numpy(np.concatenate(parts + occ).view(np.uint8).copy())

    def pack(self, kc, below, above):
        self.kc = kc
        empty = self.rows[1] <= self.rows[0]
        coarse = self._coarse(kc)
        if coarse is not None and empty:
            coarse.zero_()
        down = self._rows(kc, "down") if below and not empty and kc < self.lv else None
        up = self._rows(kc, "up") if above and not empty and kc < self.lv else None
        return coarse, down, up

    def recv_buffers(self, kc):
        n = self._rows(kc, "down").numel() if kc < self.lv else 0
        return torch.zeros(n, dtype=torch.uint8), torch.zeros(n, dtype=torch.uint8)

    def unpack(self, kc, coarse_all, world, from_below, from_above):
        lo, hi = self.rows
        if coarse_all is not None:
            per = coarse_all.numel() // world
            for r in range(world):  # rank order
                buf = coarse_all[r * per: (r + 1) * per].numpy().view(np.float64)
                off = 0
                for k in range(2, kc + 1):
                    sz = 4**k * (self.p + 1) * 2
                    part = buf[off: off + sz].view(np.complex128).reshape(4**k, self.p + 1)
                    self.mult[k] = part.copy() if r == 0 else self.mult[k] + part
                    off += sz
                for k in range(kc + 1):
                    part = buf[off: off + 4**k].astype(np.int64)
                    self.occ[k] = part if r == 0 else self.occ[k] + part
                    off += 4**k
        for buf, which in ((from_below, "below"), (from_above, "above")):
            if buf is None:
                continue
            v = buf.numpy().view(np.float64)
            off = 0
            fine = range(max(2, kc + 1), self.lv + 1)
            for k in fine:
                mk, sft = 2**k, self.lv - k
                r0 = (lo >> sft) - 2 if which == "below" else (hi >> sft)
                sz = 2 * mk * (self.p + 1) * 2
                m = self.mult[k].reshape(mk, mk, self.p + 1)
                m[r0: r0 + 2] = v[off: off + sz].view(np.complex128).reshape(2, mk, self.p + 1)
                off += sz
            for k in fine:
                mk, sft = 2**k, self.lv - k
                r0 = (lo >> sft) - 2 if which == "below" else (hi >> sft)
                self.occ[k].reshape(mk, mk)[r0: r0 + 2] = v[off: off + 2 * mk].astype(np.int64).reshape(2, mk)
                off += 2 * mk

    def down(self, shard, config, domain, counters=True):
        lv, p = config.levels, config.order
        t = self.tree
        lo, hi = shard.rows
        mult, occ = self.mult, self.occ
        local_counts = t.counts
        t.counts = occ  # exchanged occupancy for the interaction-list emptiness test
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
