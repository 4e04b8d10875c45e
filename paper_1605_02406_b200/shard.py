"""Row-band multi-GPU driver: one band context per rank.

The grid is cut into horizontal bands of rows, one per GPU.  Per cycle the bands exchange exactly what
the method couples (include/dog.h, "row-band contexts"):

1. after predict, the particles that moved into the band below / above (16-byte records, in global
   index order) -- point-to-point with the two neighbours;
2. after the cell update, every band's fixed-point born mass (one u64 each) -- all-gather; each band
   allocates its birth slots on the global born-mass CDF (Alg. 5, A-15);
3. after the joint-CDF scan, every band's joint weight (one u64 each) -- all-gather; each band then
   produces its contiguous share [F(P'), F(P' + W_band)) of the global systematic resampling (A-24).

Philox counters use global particle / slot indices, so the bands together reproduce the whole-grid
filter bit for bit (tests/test_band_gpu.py).  The transport is torch.distributed (NCCL between GPUs,
gloo on CPU for the protocol tests); ``LocalBands`` drives several bands in one process on one device
(sequential phases, host-mediated copies: no kernel waits on another).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import dog


def band_rows(height: int, world: int) -> list[tuple[int, int]]:
    """Rows [row0, row1) of each band, bottom-up; the first height % world bands get one extra row."""
    if world < 1 or world > height:
        raise ValueError(f"cannot split {height} rows into {world} bands")
    base, extra = divmod(height, world)
    rows, r = [], 0
    for b in range(world):
        n = base + (1 if b < extra else 0)
        rows.append((r, r + n))
        r += n
    return rows


def plan_bands(row_particles, width: int, world: int, min_rows: int = 8, particle_bytes: float = 64.0,
               cell_bytes: float = 56.0) -> list[tuple[int, int]]:
    """Band rebalancing: contiguous row bands of near-equal work, from the
    particles per row.  A row costs particle_bytes per particle plus cell_bytes per cell (the
    algorithmic bytes of one cycle: 64 per particle, 56 per cell).  Boundary b is the
    first row whose cost prefix reaches b/world of the total, clamped so every band keeps at least
    min_rows rows (one-hop migration needs bands at least as tall as a cycle's motion).  Deterministic:
    every rank computes the same plan from the same counts."""
    import numpy as np
    cnt = np.asarray(row_particles, dtype=np.float64).reshape(-1)
    H = cnt.size
    if world < 1 or world * min_rows > H:
        raise ValueError(f"cannot split {H} rows into {world} bands of >= {min_rows} rows")
    cost = cnt * particle_bytes + cell_bytes * width
    prefix = np.concatenate([[0.0], np.cumsum(cost)])          # prefix[r] = cost of rows < r
    total = prefix[-1]
    bounds = [0]
    for b in range(1, world):
        r = int(np.searchsorted(prefix, total * b / world, side="left"))
        r = max(r, bounds[-1] + min_rows)
        r = min(r, H - (world - b) * min_rows)
        bounds.append(r)
    bounds.append(H)
    return [(bounds[i], bounds[i + 1]) for i in range(world)]


def neighbour_counts(counts: list[tuple[int, int]], rank: int) -> tuple[int, int]:
    """Given every band's (n_down, n_up) migrant counts, the records band `rank` receives from below
    (the lower band's n_up) and from above (the upper band's n_down)."""
    world = len(counts)
    n_lo = counts[rank - 1][1] if rank > 0 else 0
    n_hi = counts[rank + 1][0] if rank < world - 1 else 0
    return n_lo, n_hi


class DistTransport:
    """Exchanges of one band over torch.distributed (rank = band index)."""

    def __init__(self, rank: int, world: int, device: torch.device, group=None):
        self.rank, self.world, self.device, self.group = rank, world, device, group

    def counts(self, n_down: int, n_up: int) -> tuple[int, int]:
        mine = torch.tensor([n_down, n_up], dtype=torch.int64, device=self.device)
        allc = torch.empty(2 * self.world, dtype=torch.int64, device=self.device)
        dist.all_gather(list(allc.chunk(self.world)), mine, group=self.group)
        c = allc.view(self.world, 2).tolist()
        return neighbour_counts([(int(a), int(b)) for a, b in c], self.rank)

    def migrate(self, send_down: torch.Tensor, send_up: torch.Tensor, recv_lo: torch.Tensor, recv_hi: torch.Tensor):
        ops = []
        if self.rank > 0:
            if send_down.numel():
                ops.append(dist.P2POp(dist.isend, send_down, self.rank - 1, group=self.group))
            if recv_lo.numel():
                ops.append(dist.P2POp(dist.irecv, recv_lo, self.rank - 1, group=self.group))
        if self.rank < self.world - 1:
            if send_up.numel():
                ops.append(dist.P2POp(dist.isend, send_up, self.rank + 1, group=self.group))
            if recv_hi.numel():
                ops.append(dist.P2POp(dist.irecv, recv_hi, self.rank + 1, group=self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def allgather_u64(self, x: torch.Tensor, out: torch.Tensor):
        dist.all_gather(list(out.chunk(self.world)), x.reshape(1), group=self.group)

    def allgather_var(self, x: torch.Tensor) -> list[torch.Tensor]:
        """Every rank's tensor [n_r, ...] (n_r may differ; same trailing shape and dtype), in rank order."""
        n = torch.tensor([x.shape[0]], dtype=torch.int64, device=self.device)
        ns = torch.zeros(self.world, dtype=torch.int64, device=self.device)
        dist.all_gather(list(ns.chunk(self.world)), n, group=self.group)
        ns = [int(v) for v in ns.tolist()]
        m = max(ns)
        pad = torch.zeros((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=self.device)
        pad[:x.shape[0]] = x.to(self.device)
        outs = [torch.zeros_like(pad) for _ in range(self.world)]
        dist.all_gather(outs, pad, group=self.group)
        return [o[:k] for o, k in zip(outs, ns)]

    def allreduce_sum(self, x: torch.Tensor) -> torch.Tensor:
        y = x.to(self.device).clone()
        dist.all_reduce(y, group=self.group)
        return y


class ShardedFilter:
    """The filter of one rank: its band of the grid, exchanging with the neighbour ranks."""

    def __init__(self, width: int, height: int, nu: int, nu_b: int, rank: int, world: int,
                 transport: DistTransport, migrant_cap: int | None = None, **params):
        self._args = (width, height, nu, nu_b, migrant_cap or max(4096, nu // 8), params)
        self.rank = rank
        self._make(band_rows(height, world), world)
        self.t = transport
        self.world, self.rank = world, rank
        dev = transport.device
        self.mass_all = torch.zeros(world, dtype=torch.int64, device=dev)
        self.weight_all = torch.zeros(world, dtype=torch.int64, device=dev)
        self.n_far = 0

    def _make(self, rows, world):
        width, height, nu, nu_b, cap, params = self._args
        rank = self.rank
        self.rows = rows
        self.row0, self.row1 = rows[rank]
        lo_row0 = rows[rank - 1][0] if rank > 0 else self.row0
        hi_row1 = rows[rank + 1][1] if rank < world - 1 else self.row1
        self.f = dog.BandFilter(width, height, nu, nu_b, self.row0, self.row1, rank, world, lo_row0, hi_row1, cap,
                                **params)

    def rebalance(self, min_rows: int = 8) -> bool:
        """Move the band boundaries to equalise the per-band work (plan_bands over the all-reduced
        particles per row), between cycles.  The bands' states are exchanged (all-gather of particles and
        m_F rows) and each rank re-creates its band context with its new rows; the global particle order
        is unchanged, so the filter continues bit-exactly.  Returns False (nothing moved) if the plan
        keeps the current bands or the state holds particles outside the grid (an empty world)."""
        import numpy as np
        width, height = self._args[0], self._args[1]
        parts, g0 = self.f.particles()
        rows_of = np.floor(parts[:, 1]).astype(np.int64)
        if parts.shape[0] and (rows_of.min() < self.row0 or rows_of.max() >= self.row1):
            ok = 0
        else:
            ok = 1
        local = np.bincount(rows_of - 0, minlength=height)[:height] if ok and parts.shape[0] else np.zeros(height, np.int64)
        flags = self.t.allreduce_sum(torch.tensor([ok], dtype=torch.int64))
        if int(flags.item()) != self.world:
            return False
        counts = self.t.allreduce_sum(torch.from_numpy(local.astype(np.int64))).cpu().numpy()
        new_rows = plan_bands(counts, width, self.world, min_rows)
        if new_rows == self.rows:
            return False
        wb, k = self.f.w_bar_k()
        all_parts = [t.cpu().numpy() for t in self.t.allgather_var(torch.from_numpy(parts))]
        all_mf = [t.cpu().numpy() for t in self.t.allgather_var(torch.from_numpy(self.f.m_free()))]
        P = np.concatenate(all_parts, axis=0)
        MF = np.concatenate(all_mf).reshape(height, width)
        self.f.close()
        self._make(new_rows, self.world)
        r0, r1 = new_rows[self.rank]
        first = int(counts[:r0].sum())
        n = int(counts[r0:r1].sum())
        self.f.set_state(P[first:first + n], first, MF[r0:r1], wb, k)
        return True

    @classmethod
    def from_config(cls, cfg, rank: int, world: int, transport: DistTransport, **over) -> "ShardedFilter":
        kw = dict(cell_size=cfg.cell_size, seed=cfg.seed, **cfg.filter_params())
        kw.update(over)
        return cls(cfg.width, cfg.height, cfg.nu, cfg.nu_b, rank, world, transport, **kw)

    def band_of(self, meas_full: torch.Tensor) -> torch.Tensor:
        """The band's rows of a full-grid measurement tensor [H][W][2] (a contiguous view)."""
        return meas_full[self.row0:self.row1]

    def step(self, meas_band: torch.Tensor, dt: float, stream=None, doppler=None, obs=None):
        """One cycle; doppler = (doppler_band [C_band, 4], p_assoc_band [C_band]) for the Doppler branch;
        obs = obs_band [C_band, 4] for the exact PHD/MIB cycle (meas_band is then ignored)."""
        f = self.f
        f.predict(dt, stream)
        n_down, n_up, n_own, n_far = f.sizes(stream)
        self.n_far = n_far
        n_lo, n_hi = self.t.counts(n_down, n_up)
        sd, su, rl, rh = f.buffers(n_down, n_up, n_lo, n_hi, stream)
        self.t.migrate(sd, su, rl, rh)
        if obs is not None:
            mass = f.assign_exact(obs, stream)
        elif doppler is not None:
            mass = f.assign_doppler(meas_band, *doppler, stream)
        else:
            mass = f.assign(meas_band, stream)
        self.t.allgather_u64(mass, self.mass_all)
        weight = f.joint(self.mass_all, stream)
        self.t.allgather_u64(weight, self.weight_all)
        f.resample(self.weight_all, stream)


class LocalBands:
    """Several bands of one grid in one process on one device: the phases run band after band and the
    exchanges are device copies (for tests and single-GPU emulation; no kernel waits on another)."""

    def __init__(self, width: int, height: int, nu: int, nu_b: int, world: int, migrant_cap: int | None = None,
                 **params):
        self._args = (width, height, nu, nu_b, migrant_cap or max(4096, nu // 8), params)
        self.world = world
        self._make(band_rows(height, world))
        self.mass_all = torch.zeros(world, dtype=torch.int64, device="cuda")
        self.weight_all = torch.zeros(world, dtype=torch.int64, device="cuda")
        self.n_far = 0

    def _make(self, rows):
        width, height, nu, nu_b, cap, params = self._args
        world = self.world
        self.rows = rows
        self.bands = []
        for b, (r0, r1) in enumerate(rows):
            lo = rows[b - 1][0] if b > 0 else r0
            hi = rows[b + 1][1] if b < world - 1 else r1
            self.bands.append(dog.BandFilter(width, height, nu, nu_b, r0, r1, b, world, lo, hi, cap, **params))

    def rebalance(self, min_rows: int = 8, rows=None) -> bool:
        """Band rebalancing (see ShardedFilter.rebalance) for the bands of this process; `rows` forces a
        given partition instead of plan_bands'."""
        import numpy as np
        width, height = self._args[0], self._args[1]
        P, _ = self.particles()
        rows_of = np.floor(P[:, 1]).astype(np.int64)
        if P.shape[0] and (rows_of.min() < 0 or rows_of.max() >= height):
            return False
        counts = np.bincount(rows_of, minlength=height)[:height]
        new_rows = rows if rows is not None else plan_bands(counts, width, self.world, min_rows)
        if new_rows == self.rows:
            return False
        MF = np.concatenate([f.m_free() for f in self.bands]).reshape(height, width)
        wb, k = self.bands[0].w_bar_k()
        for f in self.bands:
            f.close()
        self._make(new_rows)
        for b, f in enumerate(self.bands):
            r0, r1 = new_rows[b]
            first = int(counts[:r0].sum())
            n = int(counts[r0:r1].sum())
            f.set_state(P[first:first + n], first, MF[r0:r1], wb, k)
        return True

    @classmethod
    def from_config(cls, cfg, world: int, **over) -> "LocalBands":
        kw = dict(cell_size=cfg.cell_size, seed=cfg.seed, **cfg.filter_params())
        kw.update(over)
        return cls(cfg.width, cfg.height, cfg.nu, cfg.nu_b, world, **kw)

    def step(self, meas_full: torch.Tensor, dt: float, doppler=None, obs=None):
        """One cycle of every band; doppler = (doppler [H, W, 4] or [C, 4], p_assoc [C]) full-grid; obs =
        the exact filter's full-grid observation grid [C, 4] (or [H, W, 4])."""
        B = self.bands
        for f in B:
            f.predict(dt)
        sizes = [f.sizes() for f in B]
        self.n_far = max(s[3] for s in sizes)
        counts = [(s[0], s[1]) for s in sizes]
        bufs = []
        for b, f in enumerate(B):
            n_lo, n_hi = neighbour_counts(counts, b)
            bufs.append(f.buffers(counts[b][0], counts[b][1], n_lo, n_hi))
        for b in range(self.world):                   # band b's down-migrants become band b-1's "from above"
            if b > 0:
                bufs[b - 1][3].copy_(bufs[b][0])
            if b < self.world - 1:
                bufs[b + 1][2].copy_(bufs[b][1])
        width = self._args[0]
        for b, f in enumerate(B):
            r0, r1 = self.rows[b]
            if obs is not None:
                ob = obs.reshape(-1, 4)[r0 * width:r1 * width].contiguous()
                self._dop_keep = getattr(self, "_dop_keep", []) + [ob]
                m = f.assign_exact(ob)
            elif doppler is None:
                m = f.assign(meas_full[r0:r1])
            else:
                dop = doppler[0].reshape(-1, 4)[r0 * width:r1 * width].contiguous()
                pa = doppler[1].reshape(-1)[r0 * width:r1 * width].contiguous()
                self._dop_keep = getattr(self, "_dop_keep", []) + [(dop, pa)]   # alive until resample
                m = f.assign_doppler(meas_full[r0:r1], dop, pa)
            self.mass_all[b:b + 1].copy_(m)
        for b, f in enumerate(B):
            w = f.joint(self.mass_all)
            self.weight_all[b:b + 1].copy_(w)
        for f in B:
            f.resample(self.weight_all)
        self._dop_keep = []

    def particles(self):
        """All own particles in global index order: float32 [n, 4], and each band's (first index, count)."""
        import numpy as np
        parts, spans = [], []
        for f in self.bands:
            a, g = f.particles()
            parts.append(a)
            spans.append((g, a.shape[0]))
        return np.concatenate(parts, axis=0), spans
