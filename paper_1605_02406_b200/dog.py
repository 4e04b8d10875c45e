"""Thin Python binding of libdog.so (include/dog.h) -- argument marshalling only.

Every stage of the filter cycle runs in the CUDA kernels of ``csrc/``; this module only converts
arguments (torch tensors -> device pointers, streams -> cudaStream_t) and status codes -> exceptions.
There is no CPU fallback: if the library is missing or cannot load, import fails loudly.

The C functions are re-exported under their C names (``dog_create``, ``dog_step``, ...); the
``Filter`` class is a convenience wrapper over them.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# DOG_LIB selects another in-tree build of the same library (A/B experiments, tools/ab.sh)
LIB_PATH = os.environ.get("DOG_LIB") or os.path.join(_PKG, "libdog.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libdog.so not found at {LIB_PATH}: build it with `python -m paper_1605_02406_b200.build` "
        "(or __graft_entry__.build()); there is no fallback implementation")
_lib = C.CDLL(LIB_PATH)

DOG_OK, DOG_E_INVAL, DOG_E_NOMEM, DOG_E_CUDA, DOG_E_NCCL, DOG_E_MEAS, DOG_E_STATE = 0, -1, -2, -3, -4, -5, -6
DOG_FLAG_DEBUG = 1

DEBUG_IDS = {n: i + 1 for i, n in enumerate([
    "PRED_X", "PRED_Y", "PRED_VX", "PRED_VY", "KEY", "PERM", "OFFSETS", "RHO_P", "RHO_B", "RP", "RB",
    "NB", "BIRTH_X", "BIRTH_Y", "BIRTH_VX", "BIRTH_VY", "JOINT_IDX", "SCALARS"])}


class dog_grid(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("cell_size", C.c_float), ("origin_x", C.c_float),
                ("origin_y", C.c_float)]


class dog_params(C.Structure):
    _fields_ = [("p_s", C.c_float), ("p_b", C.c_float), ("sigma_pos", C.c_float), ("sigma_vel", C.c_float),
                ("sigma_birth_vel", C.c_float), ("free_tau", C.c_float), ("occ_max", C.c_float),
                ("v_max", C.c_float)]


class dog_band(C.Structure):
    _fields_ = [("row0", C.c_int32), ("row1", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
                ("lo_row0", C.c_int32), ("hi_row1", C.c_int32), ("migrant_cap", C.c_uint32)]


_vp, _f32p = C.c_void_p, C.POINTER(C.c_float)
_u32p, _u64p, _vpp = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_void_p)
_SIGS = {
    "dog_version": ([], C.c_int),
    "dog_error_string": ([C.c_int], C.c_char_p),
    "dog_create": ([C.POINTER(dog_grid), C.c_int64, C.c_int64, C.POINTER(dog_params), C.c_uint64, C.c_uint32,
                    C.c_int, C.POINTER(C.c_int), C.POINTER(_vp)], C.c_int),
    "dog_step_sharded": ([_vp, _vpp, C.c_float, _vpp], C.c_int),
    "dog_read_cells_sharded": ([_vp, _vpp, _vpp, _vpp, _vpp, _vpp], C.c_int),
    "dog_set_bands": ([_vp, C.POINTER(C.c_int32)], C.c_int),
    "dog_get_bands": ([_vp, C.POINTER(C.c_int32), C.POINTER(C.c_int)], C.c_int),
    "dog_world": ([_vp], C.c_int),
    "dog_step": ([_vp, _vp, C.c_float, _vp], C.c_int),
    "dog_step_doppler": ([_vp, _vp, _vp, _vp, C.c_float, _vp], C.c_int),
    "dog_step_exact": ([_vp, _vp, C.c_float, _vp], C.c_int),
    "dog_step_exact_lik": ([_vp, _vp, _vp, _vp, C.c_float, _vp], C.c_int),
    "dog_step_host": ([_vp, _vp, C.c_float, _vp, _vp], C.c_int),
    "dog_step_host_async": ([_vp, _vp, C.c_float, _vp, _vp], C.c_int),
    "dog_step_host_readout": ([_vp, _vp, C.c_float, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "dog_read_cells": ([_vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "dog_sync": ([_vp, _vp], C.c_int),
    "dog_destroy": ([_vp], C.c_int),
    "dog_get_state": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp, C.POINTER(C.c_int64)], C.c_int),
    "dog_set_state": ([_vp, _vp, _vp, _vp, _vp, C.c_float, _vp, C.c_int64], C.c_int),
    "dog_get_debug": ([_vp, C.c_int, _vp, C.c_size_t], C.c_int64),
    "dog_launches_per_step": ([_vp], C.c_int),
    "dog_check_transforms": ([_vp], C.c_int),
    "dog_profile_begin": ([_vp, C.c_int], C.c_int),
    "dog_profile_end": ([_vp, _vp, C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
    "dog_profile_stage_name": ([_vp, C.c_int], C.c_char_p),
    "dog_ego_scroll": ([_vp, C.c_double, C.c_double, C.POINTER(C.c_int32), C.POINTER(C.c_int32), _vp], C.c_int),
    "dog_get_origin": ([_vp, C.POINTER(C.c_double), C.POINTER(C.c_double)], C.c_int),
    "dog_ego_residual": ([_vp, C.POINTER(C.c_double), C.POINTER(C.c_double)], C.c_int),
    "dog_eval_cells": ([_vp, _vp, _vp, _vp, C.c_int, _vp, _vp, _vp, C.c_int, _vp, _vp, _vp, _vp], C.c_int),
    "dog_create_band": ([C.POINTER(dog_grid), C.c_int64, C.c_int64, C.POINTER(dog_params), C.c_uint64, C.c_uint32,
                         C.POINTER(dog_band), C.POINTER(_vp)], C.c_int),
    "dog_band_predict": ([_vp, C.c_float, _vp], C.c_int),
    "dog_band_sizes": ([_vp, _u32p, _u32p, _vp], C.c_int),
    "dog_band_outbox": ([_vp, _vpp, _vpp], C.c_int),
    "dog_band_gather": ([_vp, _vp, _vp, _vp, _vp, C.c_int, _vpp, _vpp, C.c_int, _vpp, _vpp, _vp], C.c_int),
    "dog_band_assign": ([_vp, _vp, _vpp, _vp], C.c_int),
    "dog_band_joint": ([_vp, _vp, _vpp, _vp], C.c_int),
    "dog_band_assign_doppler": ([_vp, _vp, _vp, _vp, _vpp, _vp], C.c_int),
    "dog_band_assign_exact": ([_vp, _vp, _vpp, _vp], C.c_int),
    "dog_band_resample": ([_vp, _vp, _vp], C.c_int),
    "dog_band_particles": ([_vp, _vp, C.c_uint64, _u32p, _u64p], C.c_int),
    "dog_band_set_state": ([_vp, _vp, C.c_uint32, C.c_uint64, _vp, C.c_float, C.c_int64], C.c_int),
}
DOG_MAX_STAGES = 16
for _name, (_args, _res) in _SIGS.items():
    if os.environ.get("DOG_LIB") and not hasattr(_lib, _name):   # A/B against an older build (tools/ab.sh)
        continue
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res
    globals()[_name] = _f


def check_transforms() -> tuple[int, int, int, int]:
    """include/dog.h dog_check_transforms: (ln mismatches, sqrt mismatches, packed Box-Muller mismatches,
    first failing index or 2^64-1)."""
    bad = np.zeros(4, np.uint64)
    _check(dog_check_transforms(_np_ptr(bad)), "dog_check_transforms")
    return tuple(int(b) for b in bad)


class DogError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {dog_error_string(status).decode()} ({status})")


def _check(rc: int, what: str) -> int:
    if rc < 0:
        raise DogError(rc, what)
    return rc


def _stream_ptr(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def _np_ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class Filter:
    """One DS-PHD/MIB filter (a dog_ctx) on the current CUDA device, or -- devices=[d0, d1, ...] with two
    or more entries -- a sharded context: one row band per listed device (ids may repeat), driven by
    the library with device-side exchanges (include/dog.h dog_step_sharded)."""

    def __init__(self, width: int, height: int, nu: int, nu_b: int, *, cell_size: float = 0.1,
                 p_s: float = 0.99, p_b: float = 0.02, sigma_pos: float = 0.02, sigma_vel: float = 0.8,
                 sigma_birth_vel: float = 4.0, free_tau: float = 2.0, occ_max: float = 1.0,
                 v_max: float = 0.0, seed: int = 2406, debug: bool = False, devices=None, origin=(0.0, 0.0)):
        self.width, self.height, self.nu, self.nu_b = width, height, nu, nu_b
        self.C = width * height
        g = dog_grid(width, height, cell_size, float(origin[0]), float(origin[1]))
        p = dog_params(p_s, p_b, sigma_pos, sigma_vel, sigma_birth_vel, free_tau, occ_max, v_max)
        h = _vp()
        devs = list(devices) if devices is not None else []
        ids = (C.c_int * max(1, len(devs)))(*devs)
        _check(dog_create(C.byref(g), nu, nu_b, C.byref(p), seed, DOG_FLAG_DEBUG if debug else 0, len(devs),
                          ids if devs else None, C.byref(h)), "dog_create")
        self._h = h
        self.world = dog_world(h)

    def bands(self) -> tuple[list[tuple[int, int]], list[int]]:
        """Row ranges [row0, row1) of the bands and their devices (one band for a whole-grid context)."""
        rows = (C.c_int32 * (self.world + 1))()
        devs = (C.c_int * self.world)()
        _check(dog_get_bands(self._h, rows, devs), "dog_get_bands")
        return [(rows[i], rows[i + 1]) for i in range(self.world)], list(devs)

    def set_bands(self, rows: list[tuple[int, int]]):
        """include/dog.h dog_set_bands: move the band boundaries (between cycles; the state carries over)."""
        b = [r[0] for r in rows] + [rows[-1][1]]
        _check(dog_set_bands(self._h, (C.c_int32 * len(b))(*b)), "dog_set_bands")

    def step_sharded(self, meas_bands: list, dt: float, streams: list):
        """include/dog.h dog_step_sharded: per-band measurement rows (device tensors on each band's device)
        and one stream per band."""
        assert len(meas_bands) == self.world and len(streams) == self.world
        for t in meas_bands:
            assert t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
        mp = (_vp * self.world)(*[t.data_ptr() for t in meas_bands])
        sp = (_vp * self.world)(*[_stream_ptr(s) for s in streams])
        _check(dog_step_sharded(self._h, mp, dt, sp), "dog_step_sharded")

    def read_cells_sharded(self, streams: list) -> list[dict]:
        """include/dog.h dog_read_cells_sharded: each band's readouts (tensors on the band's device)."""
        rows, devs = self.bands()
        outs = []
        for (r0, r1), d in zip(rows, devs):
            n = (r1 - r0) * self.width
            dev = torch.device("cuda", d)
            outs.append(dict(occ=torch.empty(n, device=dev), free=torch.empty(n, device=dev),
                             mean=torch.empty(n, 2, device=dev), cov=torch.empty(n, 3, device=dev)))
        arr = lambda k: (_vp * self.world)(*[o[k].data_ptr() for o in outs])
        sp = (_vp * self.world)(*[_stream_ptr(s) for s in streams])
        _check(dog_read_cells_sharded(self._h, arr("occ"), arr("free"), arr("mean"), arr("cov"), sp),
               "dog_read_cells_sharded")
        return outs

    @classmethod
    def from_config(cls, cfg, debug: bool = False, **over) -> "Filter":
        kw = dict(cell_size=cfg.cell_size, seed=cfg.seed, **cfg.filter_params())
        kw.update(over)
        return cls(cfg.width, cfg.height, cfg.nu, cfg.nu_b, debug=debug, **kw)

    def close(self):
        if getattr(self, "_h", None):
            if dog_destroy is not None:          # None during interpreter shutdown: the process frees all
                dog_destroy(self._h)
            self._h = None

    __del__ = close

    @property
    def handle(self):
        return self._h

    def launches_per_step(self) -> int:
        return _check(dog_launches_per_step(self._h), "dog_launches_per_step")

    def profile_begin(self, max_steps: int):
        _check(dog_profile_begin(self._h, max_steps), "dog_profile_begin")

    def profile_end(self) -> tuple[dict, int]:
        """Summed device ms per stage over the profiled steps, and the number of steps."""
        ms = np.zeros(DOG_MAX_STAGES, np.float32)
        ns, nst = C.c_int(), C.c_int()
        _check(dog_profile_end(self._h, _np_ptr(ms), C.byref(ns), C.byref(nst)), "dog_profile_end")
        names = [dog_profile_stage_name(self._h, i).decode() for i in range(ns.value)]
        return {n: float(ms[i]) for i, n in enumerate(names)}, nst.value

    def step(self, meas: torch.Tensor, dt: float, stream=None):
        assert meas.is_cuda and meas.dtype == torch.float32 and meas.is_contiguous()
        assert meas.numel() == 2 * self.C
        _check(dog_step(self._h, meas.data_ptr(), dt, _stream_ptr(stream)), "dog_step")

    def step_exact(self, obs: torch.Tensor, dt: float, stream=None):
        """include/dog.h dog_step_exact (NEXT-3): obs [C, 4] = (occurred, p_TP, p_FP, 0) on the device."""
        assert obs.is_cuda and obs.dtype == torch.float32 and obs.is_contiguous() and obs.numel() == 4 * self.C
        _check(dog_step_exact(self._h, obs.data_ptr(), dt, _stream_ptr(stream)), "dog_step_exact")

    def step_exact_lik(self, obs: torch.Tensor, lik: torch.Tensor, p_assoc: torch.Tensor, dt: float, stream=None):
        """include/dog.h dog_step_exact_lik (NEXT-3 with a likelihood, A-38): obs [C, 4] = (occurred, p_TP, p_FP,
        p_cl), lik [C, 4] = (u_x, u_y, v_r, sd), p_assoc [C], all on the device."""
        for t, n in ((obs, 4), (lik, 4), (p_assoc, 1)):
            assert t.is_cuda and t.dtype == torch.float32 and t.is_contiguous() and t.numel() == n * self.C
        _check(dog_step_exact_lik(self._h, obs.data_ptr(), lik.data_ptr(), p_assoc.data_ptr(), dt,
                                  _stream_ptr(stream)), "dog_step_exact_lik")

    def step_doppler(self, meas: torch.Tensor, doppler: torch.Tensor, p_assoc: torch.Tensor, dt: float, stream=None):
        """include/dog.h dog_step_doppler (NEXT-1): doppler [C, 4] = (u_x, u_y, v_r, sd), p_assoc [C]."""
        for t, n in ((meas, 2), (doppler, 4), (p_assoc, 1)):
            assert t.is_cuda and t.dtype == torch.float32 and t.is_contiguous() and t.numel() == n * self.C
        _check(dog_step_doppler(self._h, meas.data_ptr(), doppler.data_ptr(), p_assoc.data_ptr(), dt,
                                _stream_ptr(stream)), "dog_step_doppler")

    def step_host(self, meas_host: torch.Tensor, dt: float, occ_host: torch.Tensor | None = None, stream=None):
        assert not meas_host.is_cuda and meas_host.dtype == torch.float32 and meas_host.is_contiguous()
        occ_ptr = occ_host.data_ptr() if occ_host is not None else None
        _check(dog_step_host(self._h, meas_host.data_ptr(), dt, occ_ptr, _stream_ptr(stream)), "dog_step_host")

    def step_host_async(self, meas_host: torch.Tensor, dt: float, occ_host: torch.Tensor | None = None,
                        stream=None):
        """Pipelined host entry (include/dog.h): complete after sync(); use pinned tensors."""
        assert not meas_host.is_cuda and meas_host.dtype == torch.float32 and meas_host.is_contiguous()
        occ_ptr = occ_host.data_ptr() if occ_host is not None else None
        _check(dog_step_host_async(self._h, meas_host.data_ptr(), dt, occ_ptr, _stream_ptr(stream)),
               "dog_step_host_async")

    def step_host_readout(self, meas_host: torch.Tensor, dt: float, out: dict | None = None, stream=None):
        """Pipelined host entry with the full readout (include/dog.h dog_step_host_readout): out holds pinned
        host tensors occ [C], free [C], mean [C, 2], cov [C, 3] (any subset); complete after sync()."""
        assert not meas_host.is_cuda and meas_host.dtype == torch.float32 and meas_host.is_contiguous()
        out = out or {}
        ptr = lambda k: out[k].data_ptr() if k in out and out[k] is not None else None
        _check(dog_step_host_readout(self._h, meas_host.data_ptr(), dt, ptr("occ"), ptr("free"), ptr("mean"),
                                     ptr("cov"), _stream_ptr(stream)), "dog_step_host_readout")

    def ego_scroll(self, dx: float, dy: float, stream=None) -> tuple[int, int]:
        """Ego-motion compensation between cycles (include/dog.h); the applied shift in cells."""
        sx, sy = C.c_int32(), C.c_int32()
        _check(dog_ego_scroll(self._h, float(dx), float(dy), C.byref(sx), C.byref(sy), _stream_ptr(stream)),
               "dog_ego_scroll")
        return sx.value, sy.value

    def origin(self) -> tuple[float, float]:
        """include/dog.h dog_get_origin: world metres of cell (0, 0)'s lower-left corner, moved by ego scrolls."""
        ox, oy = C.c_double(), C.c_double()
        _check(dog_get_origin(self._h, C.byref(ox), C.byref(oy)), "dog_get_origin")
        return ox.value, oy.value

    def ego_residual(self) -> tuple[float, float]:
        rx, ry = C.c_double(), C.c_double()
        _check(dog_ego_residual(self._h, C.byref(rx), C.byref(ry)), "dog_ego_residual")
        return rx.value, ry.value

    def evaluate(self, labels: torch.Tensor | None = None, mask: torch.Tensor | None = None, thresholds=(),
                 mean: torch.Tensor | None = None, cov: torch.Tensor | None = None, valid: torch.Tensor | None = None,
                 stream=None, fetch: bool = True, m: torch.Tensor | None = None) -> dict:
        """Evaluation workload (NEXT-4, include/dog.h dog_eval_cells) on the filter's last readouts, or on
        the given device readouts (mean [C,2], cov [C,3], valid u8 [C]).  Returns the per-cell Mahalanobis
        distance (device), per-threshold (TP, FN, FP, TN) and the cluster sums.  fetch=False leaves the
        reductions on the device (no host synchronisation; counts/sums are returned as None)."""
        dev = torch.device("cuda", torch.cuda.current_device())
        if m is None:
            m = torch.empty(self.C, dtype=torch.float32, device=dev)
        thr = np.ascontiguousarray(thresholds, np.float32).reshape(-1)
        counts = np.zeros((max(thr.size, 1), 4), np.uint64)
        sums = np.zeros(5, np.float64)
        ptr = lambda t: None if t is None else t.data_ptr()
        own = mean is None
        _check(dog_eval_cells(self._h, ptr(mean), ptr(cov), ptr(valid), 1 if own else 0, ptr(labels), ptr(mask),
                              _np_ptr(thr) if thr.size else None, int(thr.size), m.data_ptr(),
                              _np_ptr(counts) if fetch else None, _np_ptr(sums) if fetch else None,
                              _stream_ptr(stream)), "dog_eval_cells")
        if not fetch:
            return {"m": m, "counts": None, "sums": None}
        return {"m": m, "counts": counts[:thr.size], "sums": sums}

    def sync(self, stream=None) -> int:
        return dog_sync(self._h, _stream_ptr(stream))

    def read_cells(self, stream=None, check: bool = True) -> dict:
        dev = torch.device("cuda", torch.cuda.current_device())
        out = dict(occ=torch.empty(self.C, device=dev), free=torch.empty(self.C, device=dev),
                   mean=torch.empty(self.C, 2, device=dev), cov=torch.empty(self.C, 3, device=dev))
        rc = dog_read_cells(self._h, out["occ"].data_ptr(), out["free"].data_ptr(), out["mean"].data_ptr(),
                            out["cov"].data_ptr(), _stream_ptr(stream))
        if check:
            _check(rc, "dog_read_cells")
        out["status"] = rc
        return out

    def get_state(self) -> dict:
        nu = self.nu
        x, y, vx, vy = (np.zeros(nu, np.float32) for _ in range(4))
        mf = np.zeros(self.C, np.float32)
        wb = np.zeros(1, np.float32)
        k = C.c_int64()
        _check(dog_get_state(self._h, _np_ptr(x), _np_ptr(y), _np_ptr(vx), _np_ptr(vy), _np_ptr(wb), _np_ptr(mf),
                             C.byref(k)), "dog_get_state")
        return dict(x=x, y=y, vx=vx, vy=vy, w_bar=wb[0], m_free=mf, k=k.value)

    def set_state(self, x, y, vx, vy, w_bar: float, m_free, k: int):
        arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in (x, y, vx, vy, m_free)]
        assert all(a.size == self.nu for a in arrs[:4]) and arrs[4].size == self.C
        _check(dog_set_state(self._h, *[_np_ptr(a) for a in arrs[:4]], float(w_bar), _np_ptr(arrs[4]), int(k)),
               "dog_set_state")

    _DT = {"KEY": np.uint32, "PERM": np.uint32, "OFFSETS": np.uint32, "RP": np.uint64, "RB": np.uint64,
           "NB": np.uint32, "JOINT_IDX": np.uint32, "SCALARS": np.uint64}

    def debug(self, name: str) -> np.ndarray:
        n = {"OFFSETS": self.C + 1, "SCALARS": 8}.get(name)
        if n is None:
            if name.startswith("PRED") or name in ("KEY", "PERM", "JOINT_IDX"):
                n = self.nu
            elif name.startswith("BIRTH"):
                n = self.nu_b
            else:
                n = self.C
        a = np.zeros(n, self._DT.get(name, np.float32))
        _check(dog_get_debug(self._h, DEBUG_IDS[name], _np_ptr(a), a.nbytes), f"dog_get_debug({name})")
        return a

    def scalars(self) -> dict:
        s = self.debug("SCALARS")
        return dict(W=int(s[0]), U=int(s[1]), A=int(s[2]), meas_bad=int(s[3]),
                    w_pred=np.uint32(s[4]).view(np.float32), w_bar=np.uint32(s[5]).view(np.float32),
                    k=int(s[6]), n_in=int(s[7]))


class DeviceArray:
    """A zero-copy torch view of device memory the library owns (``__cuda_array_interface__``)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}

    @staticmethod
    def tensor(ptr: int, n: int, dtype: torch.dtype) -> torch.Tensor:
        ts = {torch.float32: "<f4", torch.int64: "<i8", torch.uint8: "|u1"}[dtype]
        if n == 0:
            return torch.empty(0, dtype=dtype, device="cuda")
        return torch.as_tensor(DeviceArray(ptr, n, ts), device="cuda")


class BandFilter:
    """One row band of the grid (a band dog_ctx, include/dog.h); the cycle's phases map 1:1 onto the
    C calls.  The exchanges between bands are the caller's (paper_1605_02406_b200/shard.py)."""

    def __init__(self, width: int, height: int, nu: int, nu_b: int, row0: int, row1: int, rank: int, world: int,
                 lo_row0: int, hi_row1: int, migrant_cap: int, *, cell_size: float = 0.1, p_s: float = 0.99,
                 p_b: float = 0.02, sigma_pos: float = 0.02, sigma_vel: float = 0.8, sigma_birth_vel: float = 4.0,
                 free_tau: float = 2.0, occ_max: float = 1.0, v_max: float = 0.0, seed: int = 2406):
        self.width, self.height, self.nu, self.nu_b = width, height, nu, nu_b
        self.row0, self.row1, self.rank, self.world = row0, row1, rank, world
        self.C = width * (row1 - row0)
        g = dog_grid(width, height, cell_size)
        p = dog_params(p_s, p_b, sigma_pos, sigma_vel, sigma_birth_vel, free_tau, occ_max, v_max)
        b = dog_band(row0, row1, rank, world, lo_row0, hi_row1, migrant_cap)
        h = _vp()
        _check(dog_create_band(C.byref(g), nu, nu_b, C.byref(p), seed, 0, C.byref(b), C.byref(h)), "dog_create_band")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            if dog_destroy is not None:          # None during interpreter shutdown: the process frees all
                dog_destroy(self._h)
            self._h = None

    __del__ = close

    def predict(self, dt: float, stream=None):
        _check(dog_band_predict(self._h, dt, _stream_ptr(stream)), "dog_band_predict")

    def sizes(self, stream=None) -> tuple[list[int], int]:
        """Synchronising: the four migrant bucket counts (below, above, further below, further above) and
        the own particles of this cycle."""
        cnt = (C.c_uint32 * 4)()
        n = C.c_uint32()
        _check(dog_band_sizes(self._h, cnt, C.byref(n), _stream_ptr(stream)), "dog_band_sizes")
        return [int(c) for c in cnt], n.value

    def outbox(self) -> tuple[list[int], list[int]]:
        """Device pointers of the four packed migrant buckets and of their u32 counts (no sync)."""
        rec, cnt = (_vp * 4)(), (_vp * 4)()
        _check(dog_band_outbox(self._h, rec, cnt), "dog_band_outbox")
        return [int(r) for r in rec], [int(c) for c in cnt]

    def gather(self, lo_near, hi_near, lo_far=(), hi_far=(), stream=None):
        """include/dog.h dog_band_gather: each source is (records device pointer, u32 count device pointer);
        lo_near / hi_near None at the grid edges."""
        lf, hf = list(lo_far), list(hi_far)
        arr = lambda xs, i: (_vp * max(1, len(xs)))(*[x[i] for x in xs])
        _check(dog_band_gather(self._h, lo_near[0] if lo_near else None, lo_near[1] if lo_near else None,
                               hi_near[0] if hi_near else None, hi_near[1] if hi_near else None,
                               len(lf), arr(lf, 0), arr(lf, 1), len(hf), arr(hf, 0), arr(hf, 1),
                               _stream_ptr(stream)), "dog_band_gather")

    def assign(self, meas_band: torch.Tensor, stream=None) -> torch.Tensor:
        assert meas_band.is_cuda and meas_band.dtype == torch.float32 and meas_band.is_contiguous()
        assert meas_band.numel() == 2 * self.C
        m = _vp()
        _check(dog_band_assign(self._h, meas_band.data_ptr(), C.byref(m), _stream_ptr(stream)), "dog_band_assign")
        return DeviceArray.tensor(m.value, 1, torch.int64)

    def assign_doppler(self, meas_band: torch.Tensor, doppler_band: torch.Tensor, p_assoc_band: torch.Tensor,
                       stream=None) -> torch.Tensor:
        """include/dog.h dog_band_assign_doppler: the band's measurement, Doppler and p_A rows (device)."""
        for t, k in ((meas_band, 2), (doppler_band, 4), (p_assoc_band, 1)):
            assert t.is_cuda and t.dtype == torch.float32 and t.is_contiguous() and t.numel() == k * self.C
        m = _vp()
        _check(dog_band_assign_doppler(self._h, meas_band.data_ptr(), doppler_band.data_ptr(), p_assoc_band.data_ptr(),
                                       C.byref(m), _stream_ptr(stream)), "dog_band_assign_doppler")
        return DeviceArray.tensor(m.value, 1, torch.int64)

    def assign_exact(self, obs_band: torch.Tensor, stream=None) -> torch.Tensor:
        """include/dog.h dog_band_assign_exact: the band's rows of the exact filter's observation grid."""
        assert obs_band.is_cuda and obs_band.dtype == torch.float32 and obs_band.is_contiguous()
        assert obs_band.numel() == 4 * self.C
        m = _vp()
        _check(dog_band_assign_exact(self._h, obs_band.data_ptr(), C.byref(m), _stream_ptr(stream)),
               "dog_band_assign_exact")
        return DeviceArray.tensor(m.value, 1, torch.int64)

    def joint(self, mass_all: torch.Tensor, stream=None) -> torch.Tensor:
        assert mass_all.is_cuda and mass_all.dtype == torch.int64 and mass_all.numel() == self.world
        w = _vp()
        _check(dog_band_joint(self._h, mass_all.data_ptr(), C.byref(w), _stream_ptr(stream)), "dog_band_joint")
        return DeviceArray.tensor(w.value, 1, torch.int64)

    def resample(self, weight_all: torch.Tensor, stream=None):
        assert weight_all.is_cuda and weight_all.dtype == torch.int64 and weight_all.numel() == self.world
        _check(dog_band_resample(self._h, weight_all.data_ptr(), _stream_ptr(stream)), "dog_band_resample")

    def particles(self) -> tuple[np.ndarray, int]:
        """Own particles of the current state as float32 [n, 4] (x, y, vx, vy) and the global index of the first."""
        n, g = C.c_uint32(), C.c_uint64()
        _check(dog_band_particles(self._h, None, 0, C.byref(n), C.byref(g)), "dog_band_particles")
        a = np.zeros((n.value, 4), np.float32)
        _check(dog_band_particles(self._h, _np_ptr(a), n.value, C.byref(n), C.byref(g)), "dog_band_particles")
        return a, g.value

    def read_cells(self, stream=None, check: bool = True) -> dict:
        return Filter.read_cells(self, stream, check)

    def set_state(self, xyvv: np.ndarray, global_first: int, m_free: np.ndarray, w_bar: float, k: int):
        """include/dog.h dog_band_set_state: own particles (float32 [n, 4], global index order starting at
        global_first), m_free of the band's cells, w_bar, k."""
        a = np.ascontiguousarray(xyvv, np.float32).reshape(-1, 4)
        mf = np.ascontiguousarray(m_free, np.float32).reshape(-1)
        assert mf.size == self.C
        _check(dog_band_set_state(self._h, _np_ptr(a) if a.shape[0] else None, a.shape[0], int(global_first),
                                  _np_ptr(mf), float(w_bar), int(k)), "dog_band_set_state")

    def w_bar_k(self) -> tuple[float, int]:
        """The uniform weight of the current state and the cycle counter."""
        wb = np.zeros(1, np.float32)
        k = C.c_int64()
        _check(dog_get_state(self._h, None, None, None, None, _np_ptr(wb), None, C.byref(k)), "dog_get_state")
        return float(wb[0]), k.value

    def m_free(self) -> np.ndarray:
        mf = np.zeros(self.C, np.float32)
        _check(dog_get_state(self._h, None, None, None, None, None, _np_ptr(mf), None), "dog_get_state")
        return mf
