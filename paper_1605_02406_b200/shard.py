"""Row-band multi-GPU drivers for callers that move the band
data themselves -- one process per GPU (``ShardedFilter`` over torch.distributed) or several bands in
one process on one device (``LocalBands``).  The library's own sharded context (``dog.Filter(...,
devices=[...])``, include/dog.h dog_step_sharded) runs the same phases with device-side exchanges and
needs neither.

The grid is cut into horizontal bands of rows, one per GPU.  Per cycle the bands exchange exactly what
the method couples (include/dog.h, "row-band contexts"):

1. after predict, the particles that moved into another band (16-byte records in global index order,
   packed into four owner buckets: to the band below, above, further below, further above -- so no
   displacement is too large and nothing is dropped);
2. after the cell update, every band's fixed-point born mass (one u64 each) -- all-gather; each band
   allocates its birth slots on the global born-mass CDF (Alg. 5, A-15);
3. after the joint-CDF scan, every band's joint weight (one u64 each) -- all-gather; each band then
   produces its contiguous share [F(P'), F(P' + W_band)) of the global systematic resampling (A-24).

Philox counters use global particle / slot indices, so the bands together reproduce the whole-grid
filter bit for bit (tests/test_band_gpu.py, tests/test_sharded_gpu.py).
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


def plan_bands(row_particles, width: int, world: int, min_rows: int = 1, particle_bytes: float = 64.0,
               cell_bytes: float = 56.0) -> list[tuple[int, int]]:
    """Band rebalancing: contiguous row bands of near-equal work, from the
    particles per row.  A row costs particle_bytes per particle plus cell_bytes per cell (the
    algorithmic bytes of one cycle: 64 per particle, 56 per cell).  Boundary b is the
    first row whose cost prefix reaches b/world of the total, clamped so every band keeps at least
    min_rows rows.  Correctness does not depend on the band height (migration is owner-bucketed: a
    particle reaches its band however far it moved); min_rows only bounds how thin a band may get.
    Deterministic: every rank computes the same plan from the same counts."""
    import numpy as np
    cnt = np.asarray(row_particles, dtype=np.float64).reshape(-1)
    H = cnt.size
    min_rows = max(1, int(min_rows))
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


def sources_for(rank: int, world: int):
    """Which bucket of which band feeds band `rank` (include/dog.h dog_band_gather): (lo_near, hi_near,
    lo_far, hi_far) as (band, bucket) pairs; buckets 0 below, 1 above, 2 further below, 3 further above."""
    lo_near = (rank - 1, 1) if rank > 0 else None
    hi_near = (rank + 1, 0) if rank < world - 1 else None
    lo_far = [(s, 3) for s in range(0, rank - 1)]
    hi_far = [(s, 2) for s in range(rank + 2, world)]
    return lo_near, hi_near, lo_far, hi_far


def _band_view(ptr: int, n: int) -> torch.Tensor:
    return dog.DeviceArray.tensor(ptr, 4 * n, torch.float32).view(-1, 4)


class DistTransport:
    """Exchanges of one band over torch.distributed (rank = band index).  stage_cpu=True routes every
    collective through host memory (gloo backend: protocol tests, or several processes sharing one GPU,
    where NCCL refuses duplicate devices)."""

    def __init__(self, rank: int, world: int, device: torch.device, group=None, stage_cpu: bool = False):
        self.rank, self.world, self.device, self.group = rank, world, device, group
        self.stage_cpu = stage_cpu
        self._keep = []

    @property
    def _cdev(self):
        return torch.device("cpu") if self.stage_cpu else self.device

    def all_counts(self, counts: list[int]) -> list[list[int]]:
        mine = torch.tensor(counts, dtype=torch.int64, device=self._cdev)
        allc = torch.empty(len(counts) * self.world, dtype=torch.int64, device=self._cdev)
        dist.all_gather(list(allc.chunk(self.world)), mine, group=self.group)
        return allc.view(self.world, len(counts)).tolist()

    def _p2p(self, sends, recvs):
        ops = [dist.P2POp(dist.isend, t, peer, group=self.group) for t, peer in sends if t.numel()]
        ops += [dist.P2POp(dist.irecv, t, peer, group=self.group) for t, peer in recvs if t.numel()]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def exchange_buckets(self, out: list, counts: list[int], ok: int = 1):
        """The communication of the migrant exchange: `out` are this band's four buckets ([n_d, 4] f32
        tensors on the transport's collective device; 0 below, 1 above, 2 further below, 3 further above).
        Returns the sources of this band in dog_band_gather's order as (kind, records [n, 4], n): "lo" /
        "hi" near buckets of the neighbours (point to point), then "lof" / "hif" far buckets of the other
        bands in band order (padded all-gathers, only when some band has any).  Raises on every rank if
        any rank reports ok = 0."""
        r, w = self.rank, self.world
        allc = self.all_counts(list(counts) + [ok])
        if any(c[4] == 0 for c in allc):
            raise dog.DogError(dog.DOG_E_NOMEM, "migrant exchange (a band exceeded its migrant capacity)")
        cdev = self._cdev
        recv_lo = torch.empty(allc[r - 1][1] if r > 0 else 0, 4, device=cdev)
        recv_hi = torch.empty(allc[r + 1][0] if r < w - 1 else 0, 4, device=cdev)
        sends = ([(out[0], r - 1)] if r > 0 else []) + ([(out[1], r + 1)] if r < w - 1 else [])
        recvs = ([(recv_lo, r - 1)] if r > 0 else []) + ([(recv_hi, r + 1)] if r < w - 1 else [])
        self._p2p(sends, recvs)
        far = {}
        for d in (2, 3):
            m = max(c[d] for c in allc)
            if m == 0:
                continue
            pad = torch.zeros(m, 4, device=cdev)
            pad[:counts[d]] = out[d]
            gathered = [torch.empty(m, 4, device=cdev) for _ in range(w)]
            dist.all_gather(gathered, pad, group=self.group)
            far[d] = gathered
        lo_near, hi_near, lo_far, hi_far = sources_for(r, w)
        srcs = [("lo", recv_lo, recv_lo.shape[0])] if lo_near else []
        srcs += [("hi", recv_hi, recv_hi.shape[0])] if hi_near else []
        for kind, lst in (("lof", lo_far), ("hif", hi_far)):
            for b, d in lst:
                n = allc[b][d]
                srcs.append((kind, far[d][b][:n] if d in far else torch.empty(0, 4, device=cdev), n))
        return srcs

    def migrate(self, f, stream=None):
        """Move this band's migrant buckets to their owners and assemble the band's local array
        (dog_band_gather).  One host synchronisation: the bucket counts size the messages."""
        try:
            counts, _ = f.sizes(stream)
            ok = 1
        except dog.DogError:                         # overflow: every rank must fail together
            counts, ok = [0, 0, 0, 0], 0
        rec, _ = f.outbox()
        out = [_band_view(rec[d], counts[d]) for d in range(4)]
        if self.stage_cpu:
            out = [t.cpu() for t in out]
        srcs = self.exchange_buckets(out, counts, ok)
        dev = self.device
        recs = [t.to(dev).contiguous() if t.numel() else torch.empty(1, 4, device=dev) for _, t, _ in srcs]
        cnt = torch.tensor([n for _, _, n in srcs] or [0], dtype=torch.int32, device=dev)
        ptr = [(recs[i].data_ptr(), cnt.data_ptr() + 4 * i) for i in range(len(srcs))]
        pick = lambda k: [p for p, (kk, _, _) in zip(ptr, srcs) if kk == k]
        lo, hi = pick("lo"), pick("hi")
        f.gather(lo[0] if lo else None, hi[0] if hi else None, pick("lof"), pick("hif"), stream)
        self._keep = [recs, cnt]                     # alive until the gather kernel has run (stream order)

    def allgather_u64(self, x: torch.Tensor, out: torch.Tensor):
        if self.stage_cpu:
            xs = x.reshape(1).cpu()
            outs = [torch.empty(1, dtype=x.dtype) for _ in range(self.world)]
            dist.all_gather(outs, xs, group=self.group)
            out.copy_(torch.cat(outs).to(out.device))
            return
        dist.all_gather(list(out.chunk(self.world)), x.reshape(1), group=self.group)

    def allgather_var(self, x: torch.Tensor) -> list[torch.Tensor]:
        """Every rank's tensor [n_r, ...] (n_r may differ; same trailing shape and dtype), in rank order."""
        dev = self._cdev
        n = torch.tensor([x.shape[0]], dtype=torch.int64, device=dev)
        ns = torch.zeros(self.world, dtype=torch.int64, device=dev)
        dist.all_gather(list(ns.chunk(self.world)), n, group=self.group)
        ns = [int(v) for v in ns.tolist()]
        m = max(ns)
        pad = torch.zeros((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=dev)
        pad[:x.shape[0]] = x.to(dev)
        outs = [torch.zeros_like(pad) for _ in range(self.world)]
        dist.all_gather(outs, pad, group=self.group)
        return [o[:k] for o, k in zip(outs, ns)]

    def allreduce_sum(self, x: torch.Tensor) -> torch.Tensor:
        y = x.to(self._cdev).clone()
        dist.all_reduce(y, group=self.group)
        return y


class ShardedFilter:
    """The filter of one rank: its band of the grid, exchanging with the neighbour ranks."""

    def __init__(self, width: int, height: int, nu: int, nu_b: int, rank: int, world: int,
                 transport: DistTransport, migrant_cap: int | None = None, **params):
        # migrant_cap = nu (default): a band can receive every particle, so no exchange can overflow
        self._args = (width, height, nu, nu_b, min(migrant_cap or nu, (1 << 26) - 1), params)
        self.rank = rank
        self._make(band_rows(height, world), world)
        self.t = transport
        self.world, self.rank = world, rank
        dev = transport.device
        self.mass_all = torch.zeros(world, dtype=torch.int64, device=dev)
        self.weight_all = torch.zeros(world, dtype=torch.int64, device=dev)

    def _make(self, rows, world):
        width, height, nu, nu_b, cap, params = self._args
        rank = self.rank
        self.rows = rows
        self.row0, self.row1 = rows[rank]
        lo_row0 = rows[rank - 1][0] if rank > 0 else self.row0
        hi_row1 = rows[rank + 1][1] if rank < world - 1 else self.row1
        self.f = dog.BandFilter(width, height, nu, nu_b, self.row0, self.row1, rank, world, lo_row0, hi_row1, cap,
                                **params)

    def rebalance(self, min_rows: int = 1, rows=None) -> bool:
        """Move the band boundaries to equalise the per-band work (plan_bands over the all-reduced
        particles per row; `rows` forces a partition instead), between cycles.  The bands' states are exchanged (all-gather of particles and
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
        new_rows = list(rows) if rows is not None else plan_bands(counts, width, self.world, min_rows)
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
        obs = obs_band [C_band, 4] for the exact PHD/MIB cycle (meas_band is then ignored).  Every kernel
        and every exchange runs on `stream` (default: the current stream)."""
        st = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(st):
            f = self.f
            f.predict(dt, st)
            self.t.migrate(f, st)
            if obs is not None:
                mass = f.assign_exact(obs, st)
            elif doppler is not None:
                mass = f.assign_doppler(meas_band, *doppler, st)
            else:
                mass = f.assign(meas_band, st)
            self.t.allgather_u64(mass, self.mass_all)
            weight = f.joint(self.mass_all, st)
            self.t.allgather_u64(weight, self.weight_all)
            f.resample(self.weight_all, st)


class LocalBands:
    """Several bands of one grid in one process on one device: the phases run band after band and the
    exchanges are device copies (for tests and single-GPU emulation; no kernel waits on another)."""

    def __init__(self, width: int, height: int, nu: int, nu_b: int, world: int, migrant_cap: int | None = None,
                 **params):
        self._args = (width, height, nu, nu_b, min(migrant_cap or nu, (1 << 26) - 1), params)
        self.world = world
        self._make(band_rows(height, world))
        self.mass_all = torch.zeros(world, dtype=torch.int64, device="cuda")
        self.weight_all = torch.zeros(world, dtype=torch.int64, device="cuda")

    def _make(self, rows):
        width, height, nu, nu_b, cap, params = self._args
        world = self.world
        self.rows = rows
        self.bands = []
        for b, (r0, r1) in enumerate(rows):
            lo = rows[b - 1][0] if b > 0 else r0
            hi = rows[b + 1][1] if b < world - 1 else r1
            self.bands.append(dog.BandFilter(width, height, nu, nu_b, r0, r1, b, world, lo, hi, cap, **params))

    def rebalance(self, min_rows: int = 1, rows=None) -> bool:
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
        box = [f.outbox() for f in B]                 # (records, counts) device pointers of each bucket
        src = lambda t, d: (box[t][0][d], box[t][1][d])
        for b, f in enumerate(B):
            lo_near, hi_near, lo_far, hi_far = sources_for(b, self.world)
            f.gather(src(*lo_near) if lo_near else None, src(*hi_near) if hi_near else None,
                     [src(*x) for x in lo_far], [src(*x) for x in hi_far])
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
