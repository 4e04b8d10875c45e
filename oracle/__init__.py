"""CPU ORACLE of the DS-PHD/MIB filter cycle -- TEST INFRASTRUCTURE ONLY.

Thin ctypes wrapper around ``oracle/dog_oracle.c`` (plain single-threaded C, see its header).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` leg may import this package.  The product path (``paper_1605_02406_b200``) never
imports it, and it imports nothing from the product.

Paper: arXiv 1605.02406.  Readings of ambiguous passages: DESIGN.md section 3.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dog_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (A-21: no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "dog_oracle.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


class OrcParams(C.Structure):
    _fields_ = [
        ("width", C.c_int32), ("height", C.c_int32), ("cell_size", C.c_float),
        ("nu", C.c_int64), ("nu_b", C.c_int64),
        ("p_s", C.c_float), ("p_b", C.c_float), ("sigma_pos", C.c_float), ("sigma_vel", C.c_float),
        ("sigma_birth_vel", C.c_float), ("free_tau", C.c_float), ("occ_max", C.c_float),
        ("v_max", C.c_float), ("seed", C.c_uint64),
    ]


# dump ids (must match the enum in dog_oracle.h)
DUMPS = [
    "PRED_X", "PRED_Y", "PRED_VX", "PRED_VY", "KEY", "PERM", "OFFSETS", "S", "MP", "MFP", "OCC",
    "FREE", "RHO_P", "RHO_B", "RP", "RB", "NB", "BIRTH_X", "BIRTH_Y", "BIRTH_VX", "BIRTH_VY",
    "BIRTH_CELL", "MEAN", "COV", "JOINT_IDX", "SCALARS", "GFX", "GS", "NA", "RBA",
]
DUMP_ID = {n: i + 1 for i, n in enumerate(DUMPS)}


def _p(t):
    return C.POINTER(t)


def _declare(L):
    f32p, u32p, u64p = _p(C.c_float), _p(C.c_uint32), _p(C.c_uint64)
    L.orc_philox4x32_10.argtypes = [u32p, u32p, u32p]
    L.orc_u01.argtypes = [C.c_uint32]; L.orc_u01.restype = C.c_float
    L.orc_u01_open.argtypes = [C.c_uint32]; L.orc_u01_open.restype = C.c_float
    L.orc_ln_u24.argtypes = [C.c_uint32]; L.orc_ln_u24.restype = C.c_float
    L.orc_sincos_2pi_u24.argtypes = [C.c_uint32, f32p, f32p]
    L.orc_box_muller.argtypes = [C.c_uint32, C.c_uint32, f32p, f32p]
    L.orc_dempster.argtypes = [C.c_float] * 4 + [f32p, f32p]
    L.orc_birth_split.argtypes = [C.c_float] * 3 + [f32p, f32p]
    L.orc_birth_slots.argtypes = [u64p, C.c_int64, C.c_int64, u32p]; L.orc_birth_slots.restype = C.c_uint64
    L.orc_fx_bits.argtypes = [C.c_int64]; L.orc_fx_bits.restype = C.c_int
    L.orc_systematic_resample.argtypes = [u64p, C.c_int64, C.c_int64, C.c_uint32, u32p]
    L.orc_systematic_resample.restype = C.c_uint64
    L.orc_step_scalars.argtypes = [_p(OrcParams), C.c_float, f32p]
    L.orc_create.argtypes = [_p(OrcParams), _p(C.c_void_p)]; L.orc_create.restype = C.c_int
    L.orc_destroy.argtypes = [C.c_void_p]
    L.orc_set_state.argtypes = [C.c_void_p, f32p, f32p, f32p, f32p, C.c_float, f32p, C.c_int64]
    L.orc_get_state.argtypes = [C.c_void_p, f32p, f32p, f32p, f32p, f32p, f32p, _p(C.c_int64)]
    L.orc_step.argtypes = [C.c_void_p, f32p, C.c_float]; L.orc_step.restype = C.c_int
    L.orc_step_doppler.argtypes = [C.c_void_p, f32p, C.c_void_p, C.c_void_p, C.c_float]
    L.orc_step_doppler.restype = C.c_int
    L.orc_exp_spec.argtypes = [C.c_float]; L.orc_exp_spec.restype = C.c_float
    L.orc_step_exact.argtypes = [C.c_void_p, f32p, C.c_float]; L.orc_step_exact.restype = C.c_int
    L.orc_step_exact_lik.argtypes = [C.c_void_p, f32p, f32p, f32p, C.c_float]; L.orc_step_exact_lik.restype = C.c_int
    L.orc_birth_mean_lik.argtypes = [C.c_float] * 3; L.orc_birth_mean_lik.restype = C.c_float
    L.orc_exact_lik_cell.argtypes = [C.c_float] * 7 + [C.c_uint64, C.c_float, C.c_uint32, C.c_float, C.c_float,
                                                        C.c_float, f32p, f32p, f32p, f32p]
    L.orc_birth_assoc_exact.argtypes = [C.c_uint64, C.c_uint32, C.c_float, u32p, u64p]
    L.orc_exact_cell.argtypes = [C.c_float] * 6 + [f32p, f32p]
    L.orc_doppler_g.argtypes = [C.c_float] * 6; L.orc_doppler_g.restype = C.c_float
    L.orc_doppler_gfx.argtypes = [C.c_float, C.c_float]; L.orc_doppler_gfx.restype = C.c_uint32
    L.orc_doppler_Q.argtypes = [C.c_uint64, C.c_float, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32]
    L.orc_doppler_Q.restype = C.c_uint64
    L.orc_birth_assoc.argtypes = [C.c_uint64, C.c_uint32, C.c_float, u32p, u64p]
    L.orc_ego_scroll.argtypes = [C.c_void_p, C.c_double, C.c_double, _p(C.c_int32), _p(C.c_int32)]
    L.orc_ego_scroll.restype = C.c_int
    L.orc_ego_residual.argtypes = [C.c_void_p, _p(C.c_double), _p(C.c_double)]
    L.orc_eval_cells.argtypes = [C.c_int64, f32p, f32p, C.c_void_p, C.c_void_p, C.c_void_p, f32p, C.c_int, f32p,
                                 u64p, _p(C.c_double)]
    L.orc_read_cells.argtypes = [C.c_void_p, f32p, f32p, f32p, f32p]
    L.orc_get_dump.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t]
    L.orc_get_dump.restype = C.c_int64


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


# ---------------------------------------------------------------- primitives
def philox(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32); k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_ptr(c, C.c_uint32), _ptr(k, C.c_uint32), _ptr(out, C.c_uint32))
    return out


def u01(r: int) -> float:
    return lib().orc_u01(r)


def u01_open(r: int) -> float:
    return lib().orc_u01_open(r)


def ln_u24(m: int) -> float:
    return lib().orc_ln_u24(m)


def sincos_2pi_u24(n: int):
    s, c = C.c_float(), C.c_float()
    lib().orc_sincos_2pi_u24(n, C.byref(s), C.byref(c))
    return s.value, c.value


def box_muller(ra: int, rb: int):
    a, b = C.c_float(), C.c_float()
    lib().orc_box_muller(ra, rb, C.byref(a), C.byref(b))
    return a.value, b.value


def dempster(aO, aF, bO, bF):
    mo, mf = C.c_float(), C.c_float()
    lib().orc_dempster(aO, aF, bO, bF, C.byref(mo), C.byref(mf))
    return mo.value, mf.value


def birth_split(m_p, m_O, p_b):
    rb, rp = C.c_float(), C.c_float()
    lib().orc_birth_split(m_p, m_O, p_b, C.byref(rb), C.byref(rp))
    return rb.value, rp.value


def fx_bits(C_cells: int) -> int:
    """Fixed-point exponent FX of the masses for a grid of C cells (A-23)."""
    return int(lib().orc_fx_bits(int(C_cells)))


def birth_slots(Rb, nu_b: int) -> np.ndarray:
    Rb = np.ascontiguousarray(Rb, dtype=np.uint64)
    nb = np.zeros(len(Rb), np.uint32)
    lib().orc_birth_slots(_ptr(Rb, C.c_uint64), len(Rb), nu_b, _ptr(nb, C.c_uint32))
    return nb


def exp_spec(q: float) -> float:
    return lib().orc_exp_spec(q)


def exact_cell(S, occ_max, p_b, occurred, pTP, pFP):
    rp, rb = C.c_float(), C.c_float()
    lib().orc_exact_cell(S, occ_max, p_b, occurred, pTP, pFP, C.byref(rp), C.byref(rb))
    return rp.value, rb.value


def doppler_g(vx, vy, ux, uy, vr, sd) -> float:
    return lib().orc_doppler_g(vx, vy, ux, uy, vr, sd)


def doppler_gfx(g: float, gmax: float) -> int:
    return lib().orc_doppler_gfx(g, gmax)


def doppler_Q(Rp: int, pA: float, GSj: int, GS: int, j: int, n: int) -> int:
    return lib().orc_doppler_Q(Rp, pA, GSj, GS, j, n)


def birth_mean_lik(vr, sd, sigma_b) -> float:
    return lib().orc_birth_mean_lik(vr, sd, sigma_b)


def exact_lik_cell(S, occ_max, p_b, pTP, pFP, pcl, pA, GS, gmax, n, vr, sd, sigma_b):
    """A-38 cell update: (rho_p, rho_b, pAe, pi)."""
    out = [C.c_float() for _ in range(4)]
    lib().orc_exact_lik_cell(S, occ_max, p_b, pTP, pFP, pcl, pA, GS, gmax, n, vr, sd, sigma_b,
                             *[C.byref(o) for o in out])
    return tuple(o.value for o in out)


def birth_assoc_exact(Rb: int, nb: int, pi: float):
    na, ra = C.c_uint32(), C.c_uint64()
    lib().orc_birth_assoc_exact(Rb, nb, pi, C.byref(na), C.byref(ra))
    return na.value, ra.value


def birth_assoc(Rb: int, nb: int, pA: float):
    na, ra = C.c_uint32(), C.c_uint64()
    lib().orc_birth_assoc(Rb, nb, pA, C.byref(na), C.byref(ra))
    return na.value, ra.value


def systematic_resample(q, nu: int, U: int):
    q = np.ascontiguousarray(q, dtype=np.uint64)
    idx = np.zeros(nu, np.uint32)
    W = lib().orc_systematic_resample(_ptr(q, C.c_uint64), len(q), nu, U, _ptr(idx, C.c_uint32))
    return idx, W


# ---------------------------------------------------------------- the filter
@dataclass
class Params:
    width: int
    height: int
    nu: int
    nu_b: int
    cell_size: float = 0.1
    p_s: float = 0.99
    p_b: float = 0.02
    sigma_pos: float = 0.02
    sigma_vel: float = 0.8
    sigma_birth_vel: float = 4.0
    free_tau: float = 2.0
    occ_max: float = 1.0
    v_max: float = 0.0
    seed: int = 2406

    def c_struct(self) -> OrcParams:
        return OrcParams(self.width, self.height, self.cell_size, self.nu, self.nu_b, self.p_s,
                         self.p_b, self.sigma_pos, self.sigma_vel, self.sigma_birth_vel,
                         self.free_tau, self.occ_max, self.v_max, self.seed)


def eval_cells(mean, cov, valid=None, labels=None, mask=None, thresholds=()):
    """Evaluation workload (NEXT-4): per-cell Mahalanobis m (f32), per-threshold (TP, FN, FP, TN), cluster
    sums (|S|, sum mean_x, sum var_x + mean_x^2, sum mean_y, sum var_y + mean_y^2)."""
    mean = np.ascontiguousarray(mean, np.float32).reshape(-1, 2)
    cov = np.ascontiguousarray(cov, np.float32).reshape(-1, 3)
    Cn = mean.shape[0]
    u8 = lambda a: None if a is None else np.ascontiguousarray(a, np.uint8).reshape(-1)
    valid, labels, mask = u8(valid), u8(labels), u8(mask)
    thr = np.ascontiguousarray(thresholds, np.float32).reshape(-1)
    m = np.zeros(Cn, np.float32)
    counts = np.zeros((max(thr.size, 1), 4), np.uint64)
    sums = np.zeros(5, np.float64)
    vp = lambda a: None if a is None else a.ctypes.data
    lib().orc_eval_cells(Cn, _ptr(mean, C.c_float), _ptr(cov, C.c_float), vp(valid), vp(labels), vp(mask),
                         _ptr(thr, C.c_float) if thr.size else None, int(thr.size), _ptr(m, C.c_float),
                         _ptr(counts, C.c_uint64), sums.ctypes.data_as(C.POINTER(C.c_double)))
    return m, counts[:thr.size], sums


def step_scalars(p: Params, dt: float) -> np.ndarray:
    out = np.zeros(4, np.float32)
    ps = p.c_struct()
    lib().orc_step_scalars(C.byref(ps), dt, _ptr(out, C.c_float))
    return out


class Oracle:
    """The CPU oracle filter (one DS-PHD/MIB cycle per ``step``)."""

    def __init__(self, p: Params):
        self.p = p
        self.C = p.width * p.height
        h = C.c_void_p()
        ps = p.c_struct()
        rc = lib().orc_create(C.byref(ps), C.byref(h))
        if rc != 0:
            raise ValueError(f"orc_create failed: {rc}")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.orc_destroy(h)
            self._h = None

    def set_state(self, x, y, vx, vy, w_bar: float, m_free, k: int):
        a = [np.ascontiguousarray(v, dtype=np.float32) for v in (x, y, vx, vy, m_free)]
        lib().orc_set_state(self._h, *[_ptr(v, C.c_float) for v in a[:4]], C.c_float(w_bar),
                            _ptr(a[4], C.c_float), k)

    def get_state(self):
        nu, Cc = self.p.nu, self.C
        x, y, vx, vy = (np.zeros(nu, np.float32) for _ in range(4))
        mf = np.zeros(Cc, np.float32)
        wb = C.c_float(); k = C.c_int64()
        lib().orc_get_state(self._h, *[_ptr(v, C.c_float) for v in (x, y, vx, vy)], C.byref(wb),
                            _ptr(mf, C.c_float), C.byref(k))
        return dict(x=x, y=y, vx=vx, vy=vy, w_bar=np.float32(wb.value), m_free=mf, k=k.value)

    def step(self, meas: np.ndarray, dt: float) -> int:
        m = np.ascontiguousarray(meas, dtype=np.float32).reshape(-1)
        assert m.size == 2 * self.C
        return lib().orc_step(self._h, _ptr(m, C.c_float), C.c_float(dt))

    def step_doppler(self, meas: np.ndarray, dop, pA, dt: float) -> int:
        """NEXT-1 cycle: dop [C,4] = (u_x, u_y, v_r, sd), pA [C] association probability (0: none)."""
        m = np.ascontiguousarray(meas, dtype=np.float32).reshape(-1)
        assert m.size == 2 * self.C
        d = None if dop is None else np.ascontiguousarray(dop, dtype=np.float32).reshape(-1)
        a = None if pA is None else np.ascontiguousarray(pA, dtype=np.float32).reshape(-1)
        assert d is None or d.size == 4 * self.C
        assert a is None or a.size == self.C
        return lib().orc_step_doppler(self._h, _ptr(m, C.c_float), None if d is None else d.ctypes.data,
                                      None if a is None else a.ctypes.data, C.c_float(dt))

    def step_exact(self, obs, dt: float) -> int:
        """NEXT-3 exact PHD/MIB cycle: obs [C, 4] = (occurred, p_TP, p_FP, 0)."""
        o = np.ascontiguousarray(obs, dtype=np.float32).reshape(-1)
        assert o.size == 4 * self.C
        return lib().orc_step_exact(self._h, _ptr(o, C.c_float), C.c_float(dt))

    def step_exact_lik(self, obs, lik, pA, dt: float) -> int:
        """NEXT-3 exact PHD/MIB cycle with a single-object likelihood (A-38): obs [C, 4] = (occurred, p_TP,
        p_FP, p_cl), lik [C, 4] = (u_x, u_y, v_r, sd), pA [C] association probability."""
        o = np.ascontiguousarray(obs, dtype=np.float32).reshape(-1)
        d = np.ascontiguousarray(lik, dtype=np.float32).reshape(-1)
        a = np.ascontiguousarray(pA, dtype=np.float32).reshape(-1)
        assert o.size == 4 * self.C and d.size == 4 * self.C and a.size == self.C
        return lib().orc_step_exact_lik(self._h, _ptr(o, C.c_float), _ptr(d, C.c_float), _ptr(a, C.c_float),
                                        C.c_float(dt))

    def ego_scroll(self, dx: float, dy: float):
        """Ego-motion compensation (NEXT-2): (shift_x, shift_y) in cells, or None if refused."""
        sx, sy = C.c_int32(), C.c_int32()
        rc = lib().orc_ego_scroll(self._h, float(dx), float(dy), C.byref(sx), C.byref(sy))
        return None if rc != 0 else (sx.value, sy.value)

    def ego_residual(self):
        rx, ry = C.c_double(), C.c_double()
        lib().orc_ego_residual(self._h, C.byref(rx), C.byref(ry))
        return rx.value, ry.value

    def read_cells(self):
        Cc = self.C
        occ = np.zeros(Cc, np.float32); fr = np.zeros(Cc, np.float32)
        mean = np.zeros((Cc, 2), np.float32); cov = np.zeros((Cc, 3), np.float32)
        lib().orc_read_cells(self._h, *[_ptr(v, C.c_float) for v in (occ, fr, mean, cov)])
        return dict(occ=occ, free=fr, mean=mean, cov=cov)

    _DT = {
        "PRED_X": np.float32, "PRED_Y": np.float32, "PRED_VX": np.float32, "PRED_VY": np.float32,
        "KEY": np.uint32, "PERM": np.uint32, "OFFSETS": np.uint32, "S": np.float32,
        "MP": np.float32, "MFP": np.float32, "OCC": np.float32, "FREE": np.float32,
        "RHO_P": np.float32, "RHO_B": np.float32, "RP": np.uint64, "RB": np.uint64,
        "NB": np.uint32, "BIRTH_X": np.float32, "BIRTH_Y": np.float32, "BIRTH_VX": np.float32,
        "BIRTH_VY": np.float32, "BIRTH_CELL": np.uint32, "MEAN": np.float32, "COV": np.float32,
        "JOINT_IDX": np.uint32, "SCALARS": np.uint64, "GFX": np.uint32, "GS": np.uint64, "NA": np.uint32,
        "RBA": np.uint64,
    }

    def dump(self, name: str) -> np.ndarray:
        nu, nb, Cc = self.p.nu, self.p.nu_b, self.C
        n = {"OFFSETS": Cc + 1, "MEAN": 2 * Cc, "COV": 3 * Cc, "SCALARS": 8}.get(name)
        if n is None:
            if name.startswith("PRED") or name in ("KEY", "PERM", "JOINT_IDX", "GFX"):
                n = nu
            elif name.startswith("BIRTH"):
                n = nb
            else:
                n = Cc
        a = np.zeros(n, self._DT[name])
        got = lib().orc_get_dump(self._h, DUMP_ID[name], a.ctypes.data_as(C.c_void_p), a.nbytes)
        if got < 0:
            raise RuntimeError(f"dump {name} failed {got}")
        return a

    def scalars(self) -> dict:
        s = self.dump("SCALARS")
        return dict(W=int(s[0]), U=int(s[1]), A=int(s[2]), meas_bad=int(s[3]),
                    w_pred=np.uint32(s[4]).view(np.float32), w_bar=np.uint32(s[5]).view(np.float32),
                    k=int(s[6]), n_in=int(s[7]))
