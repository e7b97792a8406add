"""CPU stand-in for the per-rank device work of the slab-decomposed path (test infrastructure).

Implements the same primitives as paper_2601_01596_b200.slab_gpu.GpuSlabBackend with torch CPU
tensors and torch.fft, following the engine kernels' arithmetic (kernels.cuh hooks, k_gate_*),
so the orchestration in paper_2601_01596_b200/slab.py — transposes, collectives, decisions,
cross-rank escape repair — runs under gloo at world size > 1 on CPU and is checked against the
numpy oracle.  Half spectra are (a, b, H) complex128 (pitch P = H)."""
from __future__ import annotations

import numpy as np
import torch

from oracle import ffcz_oracle as O

KMAX = 2147483520.0


class CpuSlabBackend:
    ValidationError = O.ValidationError

    def __init__(self, n2):
        self.n2 = n2
        self.H = n2 // 2 + 1
        self.P = self.H
        self.device = torch.device("cpu")
        self.e_arr = self.dA = self.dB = None

    # -- per-point / per-component bounds (slab.py set_bounds) -----------------------------
    def set_bounds(self, e_arr, dA, dB):
        self.e_arr = None if e_arr is None else e_arr.double()
        self.dA, self.dB = dA, dB

    def half_lane(self, x):
        return x[..., : self.H].double().contiguous()

    def _E(self, E):
        return self.e_arr if self.e_arr is not None else E

    def _D(self, lanes, D):
        """(Re bound, Im bound) of a layout: tensors when per component, else the scalar."""
        if lanes is None:
            return D, D
        return lanes[0], (lanes[0] if lanes[1] is None else lanes[1])

    # -- buffers --------------------------------------------------------------------------
    def empty_like(self, t):
        return torch.empty_like(t)

    def zeros_real(self, shape):
        return torch.zeros(shape, dtype=torch.float64)

    def zeros_half(self, ab):
        return torch.zeros(tuple(ab) + (self.P,), dtype=torch.complex128)

    def zeros_moved(self, ab):
        return torch.zeros(tuple(ab) + (self.P,), dtype=torch.bool)

    # -- loop ------------------------------------------------------------------------------
    def eps0(self, orig, dec, E, fw, slack, eps_out):
        e = dec.double() - orig.double()
        eps_out.copy_(e)
        a = e.abs().reshape(-1)
        Ev = self._E(E)
        Ev = Ev.reshape(-1) if torch.is_tensor(Ev) else Ev
        b1 = torch.nonzero(a > Ev * (1.0 + 2.0 ** -20))
        b2 = torch.nonzero(a > Ev * fw * (1.0 + slack))
        return (int(b1[0]) if b1.numel() else -1), (int(b2[0]) if b2.numel() else -1)

    def fwd_local(self, x, A, N, gate=None):
        if gate is not None and int(gate[0]):
            return
        A.copy_(torch.fft.fft(torch.fft.rfft(x, dim=2), dim=1))

    def _fwd0(self, B):
        return torch.fft.fft(B, dim=0)

    def col0_check(self, B, Dw):
        V = self._fwd0(B)
        B.copy_(V)
        ar, ai = V.real.abs(), V.imag.abs()
        peak = float(torch.maximum(ar, ai).max())
        exc = float(torch.maximum(ar - Dw, ai - Dw).max())
        return peak, max(exc, 0.0)

    # device-resident loop interface (slab_gpu.GpuSlabBackend): the done flag gates the ops
    def loop_state(self):
        return {"gate": torch.zeros(2, dtype=torch.int32), "red": torch.zeros(2, dtype=torch.float64),
                "state": torch.zeros(2, dtype=torch.float64)}

    def col0_check_dev(self, B, D, fs, red, gate):
        if int(gate[0]):
            return
        V = self._fwd0(B)
        B.copy_(V)
        dre, dim_ = self._D(self.dB, D)
        ar, ai = V.real.abs(), V.imag.abs()
        peak = float(torch.maximum(ar, ai).max())
        exc = float(torch.maximum(ar - dre * fs, ai - dim_ * fs).max())
        red.copy_(torch.tensor([peak, max(exc, 0.0)], dtype=torch.float64))

    def decide(self, red, state, gate, max_iters):
        if int(gate[0]):
            return
        peak, ex = float(red[0]), float(red[1])
        if not ex > 1e-11 * peak:
            gate[1], state[1], gate[0] = 1, 0.0, 1
        elif float(state[0]) >= max_iters:
            gate[1], state[1], gate[0] = 0, ex, 1
        else:
            state[0] += 1.0

    def snapshot(self, ls):
        return int(ls["gate"][0])

    def done(self, snap):
        return bool(snap)

    def loop_result(self, ls):
        return int(ls["state"][0]), bool(int(ls["gate"][1])), float(ls["state"][1])

    def col0_clip_inv(self, B, D, fs, F_B, moved_B, first, gate=None):
        if gate is not None and int(gate[0]):
            return
        re, im = B.real, B.imag
        dre, dim_ = self._D(self.dB, D)
        dre, dim_ = dre * fs, dim_ * fs
        dre = torch.as_tensor(dre, dtype=torch.float64)
        dim_ = torch.as_tensor(dim_, dtype=torch.float64)
        cre = torch.maximum(torch.minimum(re, dre), -dre)
        cim = torch.maximum(torch.minimum(im, dim_), -dim_)
        dre, dim_ = cre - re, cim - im
        if first:
            F_B.copy_(torch.complex(0.0 + dre, 0.0 + dim_))
        moved_B |= (dre != 0) | (dim_ != 0)
        B.copy_(torch.fft.ifft(torch.complex(cre, cim), dim=0, norm="forward"))

    def _c2r(self, A, N):
        A1 = torch.fft.ifft(A, dim=1, norm="forward")
        return torch.fft.irfft(A1, n=self.n2, dim=2, norm="forward") * (1.0 / N)

    def inv_local_sclip(self, A, eps_out, N, E, fs, S, first, gate=None):
        if gate is not None and int(gate[0]):
            return
        x = self._c2r(A, N)
        Ew = torch.as_tensor(self._E(E) * fs, dtype=torch.float64)
        c = torch.maximum(torch.minimum(x, Ew), -Ew)
        d = c - x
        if first:
            S.copy_(0.0 + d)
        else:
            S.copy_(torch.where(d != 0, S + d, S))
        eps_out.copy_(c)

    def residual_s(self, eps, E, fw):
        return max(float((eps.abs() - self._E(E) * fw).max()), 0.0)

    # -- gate --------------------------------------------------------------------------------
    def eps0_plus_s(self, orig, dec, S, X):
        X.copy_((dec.double() - orig.double()) + S)

    def col0_rebuild(self, B2, delta_star, moved_B, F_B):
        V = self._fwd0(B2)
        F_B.copy_(torch.where(moved_B, delta_star - V, torch.zeros_like(V)))

    def col0_plain(self, src, dst, d):
        dst.copy_(torch.fft.fft(src, dim=0) if d < 0 else torch.fft.ifft(src, dim=0, norm="forward"))

    def gate(self, S, F_A, E, D, m, base_h):
        s = S.view(-1).numpy()
        Ev = self._E(E)
        step = np.ldexp(2.0 * (Ev.reshape(-1).numpy() if torch.is_tensor(Ev) else Ev), -m)
        nz = s != 0.0
        ovf = nz & (np.abs(s) / step > KMAX)
        keep = nz & ~ovf
        q = O._llround_exact(s / step)
        spat = np.where(keep, q.astype(np.int32).astype(np.float64) * step, np.where(ovf, s, 0.0))
        codes_s = q[keep].astype(np.int32)
        f = F_A[..., : self.H].reshape(-1).numpy()
        dre, dim_ = self._D(self.dA, D)
        lane = lambda x: x[..., : self.H].reshape(-1).numpy() if torch.is_tensor(x) else x
        fsr, fsi = np.ldexp(2.0 * lane(dre), -m), np.ldexp(2.0 * lane(dim_), -m)
        fnz = (f.real != 0.0) | (f.imag != 0.0)
        fovf = fnz & ((np.abs(f.real) / fsr > KMAX) | (np.abs(f.imag) / fsi > KMAX))
        fkeep = fnz & ~fovf
        qr, qi = O._llround_exact(f.real / fsr), O._llround_exact(f.imag / fsi)
        cur = np.where(fkeep, qr.astype(np.int32).astype(np.float64) * fsr +
                       1j * (qi.astype(np.int32).astype(np.float64) * fsi),
                       np.where(fovf, f, 0.0))
        codes_f = np.empty(2 * int(fkeep.sum()), dtype=np.int32)
        codes_f[0::2], codes_f[1::2] = qr[fkeep].astype(np.int32), qi[fkeep].astype(np.int32)
        k2 = np.arange(f.size) % self.H
        w = np.where((k2 == 0) | (2 * k2 == self.n2), 1, 2)
        freq_cur = torch.zeros_like(F_A)
        freq_cur[..., : self.H] = torch.from_numpy(cur.reshape(F_A[..., : self.H].shape))
        return {"spat_cur": torch.from_numpy(spat.reshape(S.shape).copy()),
                "freq_cur": freq_cur,
                "keep_s": keep, "keep_f": fkeep,
                "esc_s": torch.from_numpy(ovf.reshape(S.shape).copy()),
                "esc_f_h": torch.from_numpy(np.flatnonzero(fovf).astype(np.int64) + base_h),
                "codes_s": codes_s, "codes_f": codes_f,
                "act_s": int(nz.sum()), "act_f": int(w[fnz].sum())}

    def inv_local_repair_verify(self, Aw, eps_t, N, orig, dec, spat_cur, final_eps, E, esc_s,
                                corrected, eps_v):
        x = self._c2r(Aw, N)
        o, d = orig.double(), dec.double()
        sc = spat_cur
        e0 = d - o
        c = (d + sc) + x
        v = c - o
        corrected.copy_(c)
        if eps_v is not None:
            eps_v.copy_(v)
        Ev = self._E(E)
        vs = max(float((v.abs() - Ev).max()), 0.0)
        t = v if eps_v is None else (e0 + sc) + x  # eps_v None: decoder-view repair
        bad = t.abs() > Ev
        spat_cur.copy_(torch.where(bad, sc + (final_eps - t), sc))
        esc_s |= bad
        eps_t.copy_(t)
        return bool(bad.any()), vs

    def inv_local_verify(self, Aw, eps_v, N, orig, dec, spat_cur, E, corrected):
        x = self._c2r(Aw, N)
        o, d = orig.double(), dec.double()
        c = (d + spat_cur) + x
        corrected.copy_(c)
        v = c - o
        eps_v.copy_(v)
        return max(float((v.abs() - self._E(E)).max()), 0.0)

    def col0_mark(self, Bt, D):
        V = self._fwd0(Bt)
        Bt.copy_(V)
        dre, dim_ = self._D(self.dB, D)
        return (V.real.abs() > dre) | (V.imag.abs() > dim_)

    def col0_verify(self, Bv, D):
        V = self._fwd0(Bv)
        dre, dim_ = self._D(self.dB, D)
        return max(float(torch.maximum(V.real.abs() - dre, V.imag.abs() - dim_).max()), 0.0)

    # -- sparse bookkeeping ------------------------------------------------------------------
    def positions(self, viol):
        return torch.nonzero(viol.reshape(-1)).view(-1)

    def merge_sorted(self, a, b):
        return torch.unique(torch.cat([a, b]))

    def nonzero_flat(self, mask):
        return torch.nonzero(mask.reshape(-1)).view(-1)

    def take_real(self, x, idx):
        return x.reshape(-1)[idx]

    def owned_b(self, h, n0, n1, H, r, c1):
        i1 = torch.div(h, H, rounding_mode="floor") % n1
        return torch.unique(h[torch.div(i1, c1, rounding_mode="floor") == r])

    def values_at_h(self, B, h, n1, H, r, c1):
        row = torch.div(h, H, rounding_mode="floor")
        i0, i1, k2 = torch.div(row, n1, rounding_mode="floor"), row % n1, h % H
        off = (i0 * c1 + (i1 - r * c1)) * B.shape[-1] + k2
        return B.reshape(-1)[off]
