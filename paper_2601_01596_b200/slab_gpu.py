"""B200 backend of the slab-decomposed correction (paper_2601_01596_b200/slab.py): every per-rank
device step is one ffcz_cuda_slab() call of the engine (include/ffcz_cuda.h) on CUDA torch
tensors, on the context's stream (= torch's current stream, so the NCCL all-to-alls of the
orchestrator are ordered with the passes).  No CPU fallback: without the built library or a GPU
this raises."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi as capi
from .ffcz import Context, ValidationError, _check


class SlabOp(C.Structure):
    _fields_ = [("op", C.c_int32), ("dir", C.c_int32), ("first", C.c_int32),
                ("in_dtype", C.c_int32), ("m", C.c_int32), ("pad", C.c_int32),
                ("d0", C.c_uint64), ("d1", C.c_uint64), ("n2", C.c_uint64),
                ("n_total", C.c_uint64), ("e", C.c_double), ("delta", C.c_double),
                ("fscale", C.c_double), ("slack", C.c_double), ("p", C.c_void_p * 10),
                ("e_arr", C.c_void_p), ("d_re", C.c_void_p), ("d_im", C.c_void_p),
                ("rank", C.c_int32), ("world", C.c_int32)]


(EPS0, FWD_LOCAL, COL0_CHECK, COL0_CLIP_INV, COL0_PLAIN, COL0_REBUILD, COL0_MARK, COL0_VERIFY,
 INV_SCLIP, INV_REPAIR_VERIFY, INV_VERIFY, RESIDUAL_S, EPS0_PLUS_S, GATE, DECIDE,
 FWD_LOCAL_PEER, COL0_CLIP_INV_PEER) = range(17)


_E_OPS = frozenset({EPS0, INV_SCLIP, INV_REPAIR_VERIFY, INV_VERIFY, RESIDUAL_S, GATE})
_B_OPS = frozenset({COL0_CHECK, COL0_CLIP_INV, COL0_CLIP_INV_PEER, COL0_MARK, COL0_VERIFY})


def _pow2(v):
    return v > 0 and v & (v - 1) == 0


def _bits_to_bool(words, n):
    """LSB-first uint32 bitmap (device tensor) -> numpy bool[n]."""
    b = words.cpu().numpy().view(np.uint8)
    return np.unpackbits(b, bitorder="little")[:n].astype(bool)


class GpuSlabBackend:
    ValidationError = ValidationError

    def __init__(self, n2, device, ctx: Context | None = None):
        import torch
        self.torch = torch
        self.n2 = int(n2)
        self.H = self.n2 // 2 + 1
        self.lib = capi.load()
        self.P = int(self.lib.ffcz_cuda_slab_pitch(self.n2))
        self.device = torch.device(device)
        # one side stream for the engine AND the orchestrator's torch ops (transposes, sparse
        # bookkeeping), so they are ordered with each other (stream 0 would make the engine
        # create a private stream)
        self.stream = torch.cuda.Stream(self.device)
        self.ctx = ctx or Context(self.device.index or 0, self.stream.cuda_stream)
        self.e_arr = self.dA = self.dB = None
        self.swap_axes = False

    def set_axes(self, swap):
        """One-rank slab: the axis-0 ops run on axis 1 and the local ops on axis 0."""
        self.swap_axes = bool(swap)

    # -- per-point / per-component bounds (slab.py set_bounds) ----------------------------------
    def set_bounds(self, e_arr, dA, dB):
        """e_arr: (c0, n1, n2) float64 per-point E of this slab; dA / dB: (Re, Im-or-None) lanes
        in the pitched half layout of the natural slab / of the B layout."""
        torch = self.torch
        self.e_arr = None if e_arr is None else e_arr.to(torch.float64).contiguous()
        self.dA, self.dB = dA, dB

    def half_lane(self, x):
        """(c0, n1, n2) full-spectrum lane slab -> (c0, n1, P) half layout (k2 <= n2/2)."""
        torch = self.torch
        out = torch.zeros(tuple(x.shape[:2]) + (self.P,), dtype=torch.float64, device=self.device)
        out[..., : self.H] = x[..., : self.H]
        return out

    def stream_context(self):
        """Enter the backend stream (ordered after the caller's current stream) for one call."""
        import contextlib
        torch = self.torch

        @contextlib.contextmanager
        def cm():
            caller = torch.cuda.current_stream(self.device)
            self.stream.wait_stream(caller)
            with torch.cuda.stream(self.stream):
                yield
            caller.wait_stream(self.stream)
        return cm()

    # -- plumbing -----------------------------------------------------------------------------
    # which bound arrays an op reads: spatial ops the per-point E, spectrum ops the Delta lanes
    # of the layout they work in (B: axis-0 ops, A: the gate)
    def _op(self, code, shape, ptrs, gate=None, **kw):
        o = SlabOp()
        if self.e_arr is not None and code in _E_OPS:
            o.e_arr = self.e_arr.data_ptr()
        lanes = self.dB if code in _B_OPS else (self.dA if code == GATE else None)
        if lanes is not None:
            o.d_re = lanes[0].data_ptr()
            o.d_im = None if lanes[1] is None else lanes[1].data_ptr()
        o.op = code
        o.d0, o.d1 = int(shape[0]), int(shape[1])
        o.n2 = self.n2
        for k, v in kw.items():
            setattr(o, k, v)
        for i, t in enumerate(ptrs):
            o.p[i] = None if t is None else t.data_ptr()
        if gate is not None:   # device-resident loop: the op returns at once once done is set
            o.p[9] = gate.data_ptr()
        o.pad = 1 if self.swap_axes else 0   # FFCZ_SLAB_SWAP_AXES
        out = (C.c_double * 4)()
        _check(self.lib.ffcz_cuda_slab(self.ctx.handle, C.byref(o), out))
        return list(out)

    @staticmethod
    def _dtype(t):
        import torch
        return capi.FFCZ_F32 if t.dtype == torch.float32 else capi.FFCZ_F64

    def empty_like(self, t):
        return self.torch.empty_like(t)

    def zeros_real(self, shape):
        return self.torch.zeros(shape, dtype=self.torch.float64, device=self.device)

    def zeros_half(self, ab):
        return self.torch.zeros(tuple(ab) + (self.P,), dtype=self.torch.complex128,
                                device=self.device)

    def zeros_moved(self, ab):
        return self.torch.zeros(tuple(ab) + (self.P,), dtype=self.torch.uint8, device=self.device)

    def _words(self, n):
        return self.torch.zeros(((n + 31) // 32,), dtype=self.torch.int32, device=self.device)

    # -- loop ---------------------------------------------------------------------------------
    def eps0(self, orig, dec, E, fw, slack, eps_out):
        o = self._op(EPS0, orig.shape, [orig, dec, eps_out], in_dtype=self._dtype(orig), e=E,
                     fscale=fw, slack=slack)
        return int(o[0]), int(o[1])

    def fwd_local(self, x, A, N, gate=None):
        self._op(FWD_LOCAL, x.shape, [x, A], gate=gate)

    def col0_check(self, B, Dw):
        o = self._op(COL0_CHECK, B.shape, [B], delta=Dw, fscale=1.0)
        return o[0], o[1]

    def col0_clip_inv(self, B, D, fs, F_B, moved_B, first, gate=None):
        self._op(COL0_CLIP_INV, B.shape, [B, F_B, moved_B], gate=gate, delta=D, fscale=fs,
                 first=int(bool(first)))

    def inv_local_sclip(self, A, eps_out, N, E, fs, S, first, gate=None):
        self._op(INV_SCLIP, A.shape, [A, eps_out, S], gate=gate, e=E, fscale=fs, n_total=N,
                 first=int(bool(first)))

    def inv_sclip_fwd(self, A, eps_out, N, E, fs, S, first, gate=None, col=True):
        """inv_local_sclip + the forward row step in ONE row pass (C2R -> s-clip -> R2C, eps still
        written) back into A, then (col=True) the forward local pass — fwd_local(eps_out, A)
        without the eps round trip; col=False leaves the column pass to fwd_local_peer(None)."""
        self._op(INV_SCLIP, A.shape, [A, eps_out, S, A, A if col else None], gate=gate, e=E,
                 fscale=fs, n_total=N, first=int(bool(first)))

    # -- fused all-to-all: the loop's two transposes as peer stores of the passes -------------------
    def peer_ok(self, dims, W):
        """The scattering passes carry hooks (power-of-two axes 0 and 1, in [16, 4096]) and
        decode 32-bit offsets."""
        n0, n1, _ = dims
        c0, c1 = n0 // W, n1 // W
        return (W >= 2 and not self.swap_axes and _pow2(W)
                and all(_pow2(v) and 16 <= v <= 4096 for v in (n0, n1))
                and c0 * n1 * self.P < 2 ** 32 and n0 * c1 * self.P < 2 ** 32)

    def peer_setup(self, comm, dims):
        """This rank's receive buffers A (c0, n1, P) and B (n0, c1, P), exported over CUDA IPC and
        mapped by every rank; returns the state the *_peer ops and peer_close take, or None on
        every rank when some rank cannot export or map them (the loop then uses the
        all-to-alls)."""
        torch = self.torch
        n0, n1, _ = dims
        W, r = comm.size, comm.rank
        c0, c1 = n0 // W, n1 // W
        A = self.zeros_half((c0, n1))
        B = self.zeros_half((n0, c1))
        row = np.zeros(2 * 72, dtype=np.uint8)
        ok = 1
        for j, t in enumerate((A, B)):
            h = (C.c_ubyte * 64)()
            off = C.c_uint64()
            # (fails e.g. on expandable-segment allocations: then every rank takes the
            # all-to-all path, decided together below)
            if self.lib.ffcz_cuda_ipc_handle(self.ctx.handle, C.c_void_p(t.data_ptr()),
                                             C.cast(h, C.c_void_p), C.byref(off)) != 0:
                ok = 0
                break
            row[72 * j: 72 * j + 64] = np.frombuffer(bytes(h), dtype=np.uint8)
            row[72 * j + 64: 72 * j + 72] = np.frombuffer(np.uint64(off.value).tobytes(),
                                                          dtype=np.uint8)
        if comm.min_i64([ok], self.device)[0] == 0:
            return None
        dev_row = torch.as_tensor(row).view(1, -1).to(self.device)
        rows = comm.all_gather_rows(dev_row).cpu().numpy()
        opened, ptrs = [], {0: [], 1: []}
        for s in range(W):
            for j, t in enumerate((A, B)):
                if not ok:
                    break
                if s == r:
                    ptrs[j].append(t.data_ptr())
                    continue
                h = (C.c_ubyte * 64).from_buffer_copy(rows[s, 72 * j: 72 * j + 64].tobytes())
                off = int(rows[s, 72 * j + 64: 72 * j + 72].view(np.uint64)[0])
                base = C.c_void_p()
                if self.lib.ffcz_cuda_ipc_open(self.ctx.handle, C.cast(h, C.c_void_p),
                                               C.byref(base)) != 0:
                    ok = 0   # e.g. no peer access between these GPUs
                    break
                opened.append(base.value)
                ptrs[j].append(base.value + off)
        if comm.min_i64([ok], self.device)[0] == 0:
            self.peer_close({"opened": opened})
            return None
        return {"A": A, "B": B, "W": W, "r": r, "opened": opened,
                # each op scatters into the OTHER layout's buffers
                "to_A": torch.tensor(ptrs[0], dtype=torch.int64, device=self.device),
                "to_B": torch.tensor(ptrs[1], dtype=torch.int64, device=self.device)}

    def peer_close(self, peer):
        for base in peer["opened"]:
            _check(self.lib.ffcz_cuda_ipc_close(self.ctx.handle, C.c_void_p(base)))
        peer["opened"] = []

    def fwd_local_peer(self, x, peer, gate=None):
        """R2C rows + forward axis 1 of x into peer A, scattered into every rank's B."""
        A = peer["A"]   # (x None: A's rows are already transformed, inv_sclip_fwd(col=False))
        self._op(FWD_LOCAL_PEER, A.shape, [x, A] + [None] * 6 + [peer["to_B"]], gate=gate,
                 rank=peer["r"], world=peer["W"])

    def col0_clip_inv_peer(self, D, fs, F_B, moved_B, first, peer, gate=None):
        """project_onto_fcube + inverse axis 0 of peer B, scattered into every rank's A."""
        B = peer["B"]
        self._op(COL0_CLIP_INV_PEER, B.shape, [B, F_B, moved_B] + [None] * 5 + [peer["to_A"]],
                 gate=gate, delta=D, fscale=fs, first=int(bool(first)), rank=peer["r"],
                 world=peer["W"])

    # -- device-resident loop: decisions on the device, the host only waits on events ------------
    def loop_state(self):
        torch = self.torch
        return {"gate": torch.zeros(2, dtype=torch.int32, device=self.device),    # done, conv.
                "red": torch.zeros(2, dtype=torch.float64, device=self.device),   # peak, excess
                "state": torch.zeros(2, dtype=torch.float64, device=self.device),  # passes, res.
                "host": [torch.zeros(2, dtype=torch.int32, pin_memory=True) for _ in range(2)],
                "slot": 0}

    def col0_check_dev(self, B, D, fs, red, gate):
        self._op(COL0_CHECK, B.shape, [B, red], gate=gate, delta=D, fscale=fs)

    def decide(self, red, state, gate, max_iters):
        self._op(DECIDE, (1, 1), [red, state], gate=gate, n_total=int(max_iters))

    def snapshot(self, ls):
        """Queue an async copy of the done flag; returns a handle for done()."""
        h = ls["host"][ls["slot"]]
        ls["slot"] ^= 1
        h.copy_(ls["gate"], non_blocking=True)
        ev = self.torch.cuda.Event()
        ev.record(self.torch.cuda.current_stream(self.device))
        return (ev, h)

    def done(self, snap):
        ev, h = snap
        ev.synchronize()
        return bool(h[0].item())

    def loop_result(self, ls):
        """(passes, converged, residual_f) after the loop (one sync)."""
        st, g = ls["state"].cpu().tolist(), ls["gate"].cpu().tolist()
        return int(st[0]), bool(g[1]), float(st[1])

    def residual_s(self, eps, E, fw):
        return self._op(RESIDUAL_S, eps.shape, [eps], e=E, fscale=fw)[0]

    # -- gate ---------------------------------------------------------------------------------
    def eps0_plus_s(self, orig, dec, S, X):
        self._op(EPS0_PLUS_S, orig.shape, [orig, dec, S, X], in_dtype=self._dtype(orig))

    def col0_rebuild(self, B2, delta_star, moved_B, F_B):
        self._op(COL0_REBUILD, B2.shape, [B2, delta_star, moved_B, F_B])

    def col0_plain(self, src, dst, d):
        self._op(COL0_PLAIN, src.shape, [src, dst], dir=int(d))

    def gate(self, S, F_A, E, D, m, base_h):
        torch = self.torch
        c0, n1, n2 = S.shape
        N, Nc = c0 * n1 * n2, c0 * n1 * self.H
        spat, freq = torch.empty_like(S), torch.empty_like(F_A)
        ks, es, kf, ef = self._words(N), self._words(N), self._words(Nc), self._words(Nc)
        cs = torch.empty((N,), dtype=torch.int32, device=self.device)
        cf = torch.empty((2 * Nc,), dtype=torch.int32, device=self.device)
        o = self._op(GATE, S.shape, [S, F_A, spat, freq, ks, es, kf, ef, cs, cf], e=E, delta=D,
                     m=int(m))
        ks_n, kf_n = int(o[2]), int(o[3])
        # flags stay LSB-first bitmaps and codes stay on the device (flags_to_bool for checks)
        return {"spat_cur": spat, "freq_cur": freq, "keep_s": ks, "keep_f": kf, "esc_s": es,
                "esc_f_h": self._bit_positions(ef) + base_h,
                "codes_s": cs[:ks_n], "codes_f": cf[: 2 * kf_n],
                "act_s": int(o[0]), "act_f": int(o[1])}

    @staticmethod
    def flags_to_bool(words, n):
        return _bits_to_bool(words, n)

    def inv_local_repair_verify(self, Aw, eps_t, N, orig, dec, spat_cur, final_eps, E, esc_s,
                                corrected, eps_v):
        o = self._op(INV_REPAIR_VERIFY, Aw.shape,
                     [Aw, eps_t, orig, dec, spat_cur, final_eps, esc_s, corrected, eps_v],
                     in_dtype=self._dtype(orig), e=E, n_total=N)
        return bool(o[0]), o[1]

    def inv_local_verify(self, Aw, eps_v, N, orig, dec, spat_cur, E, corrected):
        o = self._op(INV_VERIFY, Aw.shape, [Aw, eps_v, orig, dec, spat_cur, corrected],
                     in_dtype=self._dtype(orig), e=E, n_total=N)
        return o[1]

    def col0_mark(self, Bt, D):
        w = self._words(Bt.numel())
        self._op(COL0_MARK, Bt.shape, [Bt, w], delta=D)
        return w

    def col0_verify(self, Bv, D):
        return self._op(COL0_VERIFY, Bv.shape, [Bv], delta=D)[0]

    # -- sparse bookkeeping (small index sets) -------------------------------------------------
    def _bit_positions(self, words):
        torch = self.torch
        w = words.view(-1)
        nz = torch.nonzero(w).view(-1)
        if nz.numel() == 0:
            return torch.zeros(0, dtype=torch.int64, device=self.device)
        bits = (w[nz].to(torch.int64).unsqueeze(1) >> torch.arange(32, device=self.device)) & 1
        r, b = torch.nonzero(bits, as_tuple=True)
        return nz[r] * 32 + b

    def positions(self, viol):
        return self._bit_positions(viol)

    def merge_sorted(self, a, b):
        return self.torch.unique(self.torch.cat([a, b]))

    def nonzero_flat(self, mask):
        return self._bit_positions(mask)

    def take_real(self, x, idx):
        return x.reshape(-1)[idx]

    def owned_b(self, h, n0, n1, H, r, c1):
        torch = self.torch
        i1 = torch.div(h, H, rounding_mode="floor") % n1
        return torch.unique(h[torch.div(i1, c1, rounding_mode="floor") == r])

    def values_at_h(self, B, h, n1, H, r, c1):
        torch = self.torch
        row = torch.div(h, H, rounding_mode="floor")
        i0, i1, k2 = torch.div(row, n1, rounding_mode="floor"), row % n1, h % H
        off = (i0 * c1 + (i1 - r * c1)) * B.shape[-1] + k2
        return B.reshape(-1)[off]


def correct_slab_gpu(orig_slab, dec_slab, dims, E, Delta, m=16, max_iters=1000, group=None,
                     ctx: Context | None = None):
    """ffcz::correct of a volume slab-decomposed along axis 0 across the ranks of `group`
    (torch.distributed, NCCL): this rank passes its (n0/W, n1, n2) CUDA slab of both fields."""
    from .slab import Comm, correct_slab
    be = GpuSlabBackend(dims[2], orig_slab.device, ctx)
    return correct_slab(be, Comm(group), dims, orig_slab, dec_slab, E, Delta, m, max_iters)
