"""Slab-decomposed correction of ONE volume across ranks (BASELINE configs 4/5).

The reference's ``ffcz::correct`` (proj/core/src/pipeline.cpp:26-178) on a field split into
slabs along axis 0: rank r holds planes i0 in [r*c0, (r+1)*c0).  The 3-D transform is
separable, so every iteration of ``alternating_projection`` (projection.cpp:96-126) becomes

    A (c0, n1, P) natural slab  --R2C rows, FFT axis 1 (local)-->  A
    A --all-to-all #1-->  B (n0, c1, P): rank r holds i1 in [r*c1, (r+1)*c1), all i0
    B --FFT axis 0 + check_convergence (local) + all-reduce(max) of (peak, excess)-->  decision
    B --project_onto_fcube + inverse axis 0 (local)-->  B  --all-to-all #2-->  A
    A --inverse axis 1, C2R, project_onto_scube (local)-->  eps

so the frequency-domain state (F, the clip map, the converged spectrum delta_star) lives in the
B layout and the spatial state (eps, S, spat_cur) in the natural slab.  The FP64 gate follows
pipeline.cpp:46-176 in the same two layouts: quantisation and compaction on natural slabs (so
each rank's flag bits / codes are a contiguous range of the global half-grid order), escape
repair rounds with the frequency side in B; the conjugate partners of the k2 = 0 / n2/2 planes
(pipeline.cpp:149-151) may live on another rank, so those few repairs are exchanged with one
all-gather per round.

The per-rank device work goes through a backend (``GpuSlabBackend`` = the B200 engine's slab
C-ABI; the CPU test suite drives the same orchestration with a torch stand-in under gloo).  The
collectives are torch.distributed (NCCL over NVLink on the box).  Every decision the reference
makes is made identically on every rank from all-reduced values, so the control flow equals the
single-volume path's.
"""
from __future__ import annotations

import os
import sys

from dataclasses import dataclass, field

import numpy as np

KMAX_ITER_TOL = 1e-11           # projection.cpp:40
MAX_ESCAPE_ROUNDS = 32          # pipeline.cpp:15


class Comm:
    """The collectives the slab path needs, over torch.distributed (or a single process)."""

    def __init__(self, group=None, stage_cpu: bool = False):
        """stage_cpu: run the collectives on host copies (gloo) — lets several ranks share one
        GPU in the tests; the product path uses NCCL on device tensors."""
        import torch.distributed as dist
        self.dist = dist
        self.on = dist.is_available() and dist.is_initialized()
        self.group = group
        self.size = dist.get_world_size(group) if self.on else 1
        self.rank = dist.get_rank(group) if self.on else 0
        self.stage_cpu = stage_cpu

    def all_to_all(self, out, inp):
        if self.size == 1:
            out.copy_(inp)
            return
        import torch
        dst = out
        if self.stage_cpu:
            inp, out = inp.cpu(), torch.empty(out.shape, dtype=out.dtype)
        if inp.is_complex():   # collectives move bytes: complex128 as (re, im) float64 pairs
            self.dist.all_to_all_single(torch.view_as_real(out), torch.view_as_real(inp),
                                        group=self.group)
        else:
            self.dist.all_to_all_single(out, inp, group=self.group)
        if dst is not out:
            dst.copy_(out)

    def barrier_dev(self):
        """Order every rank's device work so far before any rank's next op (the fused all-to-all's
        receive buffers): a one-element all-reduce on the stream (NCCL), or a host barrier after a
        device sync when the collectives are staged on the host."""
        if self.size == 1:
            return
        import torch
        if self.stage_cpu:
            torch.cuda.synchronize()
            self.dist.barrier(group=self.group)
            return
        if getattr(self, "_tick", None) is None:
            self._tick = torch.zeros(1, dtype=torch.int32, device=torch.cuda.current_device())
        self.dist.all_reduce(self._tick, group=self.group)

    def _reduce(self, t, op):
        if self.size > 1:
            if self.stage_cpu:
                h = t.cpu()
                self.dist.all_reduce(h, op=op, group=self.group)
                t.copy_(h)
            else:
                self.dist.all_reduce(t, op=op, group=self.group)
        return t

    def max_f64_(self, t):
        """In-place all-reduce(max) of a float64 device tensor, no host sync (stream ordered)."""
        return self._reduce(t, self.dist.ReduceOp.MAX)

    def max_f64(self, values, device):
        import torch
        t = torch.tensor(list(values), dtype=torch.float64, device=device)
        return self._reduce(t, self.dist.ReduceOp.MAX).tolist()

    def min_i64(self, values, device):
        import torch
        t = torch.tensor(list(values), dtype=torch.int64, device=device)
        return self._reduce(t, self.dist.ReduceOp.MIN).tolist()

    def sum_i64(self, values, device):
        import torch
        t = torch.tensor(list(values), dtype=torch.int64, device=device)
        return self._reduce(t, self.dist.ReduceOp.SUM).tolist()

    def all_gather_rows(self, t):
        """Concatenate a (k_r, w) tensor of every rank (variable k_r) in rank order."""
        import torch
        if self.size == 1:
            return t
        if self.stage_cpu and t.device.type != "cpu":
            return self.all_gather_rows(t.cpu()).to(t.device)
        k = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        ks = [torch.zeros_like(k) for _ in range(self.size)]
        self.dist.all_gather(ks, k, group=self.group)
        kmax = max(int(x.item()) for x in ks)
        pad = torch.zeros((kmax,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        outs = [torch.zeros_like(pad) for _ in range(self.size)]
        self.dist.all_gather(outs, pad, group=self.group)
        return torch.cat([o[: int(kk.item())] for o, kk in zip(outs, ks)])


class EscapeList:
    """The global escape list in std::map order (spatial by index, then frequency by half index)
    as columns; iterating / indexing yields (is_freq, global index, re, im) tuples.  (Tuples per
    element cost 0.19 s for the 263 K escapes of 1024^3 config 4; the columns cost nothing.)"""

    def __init__(self, sp, fr):
        self.sp_index = sp[:, 0].astype(np.int64)
        self.sp_value = np.ascontiguousarray(sp[:, 1])
        self.fr_index = fr[:, 0].astype(np.int64)
        self.fr_re = np.ascontiguousarray(fr[:, 1])
        self.fr_im = np.ascontiguousarray(fr[:, 2])

    def __len__(self):
        return len(self.sp_index) + len(self.fr_index)

    def __getitem__(self, i):
        if i < 0:
            i += len(self)
        ns = len(self.sp_index)
        if i < ns:
            return (False, int(self.sp_index[i]), float(self.sp_value[i]), 0.0)
        j = i - ns
        if j >= len(self.fr_index):
            raise IndexError(i)
        return (True, int(self.fr_index[j]), float(self.fr_re[j]), float(self.fr_im[j]))

    def __iter__(self):
        yield from zip([False] * len(self.sp_index), self.sp_index.tolist(),
                       self.sp_value.tolist(), [0.0] * len(self.sp_index))
        yield from zip([True] * len(self.fr_index), self.fr_index.tolist(), self.fr_re.tolist(),
                       self.fr_im.tolist())


@dataclass
class SlabResult:
    """This rank's part of ffcz::CorrectionResult (pipeline.hpp:11-16).  Flags and codes cover
    the rank's contiguous range of the global order; escapes are global (every rank)."""
    iterations: int
    converged: bool
    residual_f: float
    residual_s: float
    active_spatial: int
    active_frequency: int
    verify_ok: bool
    verify_max_spatial_excess: float
    verify_max_freq_excess: float
    escape_rounds: int
    spatial_flags: object            # this rank's c0*n1*n2 flags (backend form: bool / bitmap)
    frequency_flags: object          # this rank's c0*n1*H half-grid flags
    spatial_codes: object            # int32, ascending index order (backend tensor / array)
    frequency_codes: object          # int32, interleaved (Re, Im)
    escapes: object = field(default_factory=list)  # EscapeList: (is_freq, index, re, im), map order
    corrected: object = None         # this rank's FP64 corrected slab (backend tensor)


def _transpose_ab(be, comm, A, n0, c0, c1):
    """A (c0, n1, P) -> B (n0, c1, P): all-to-all #1."""
    W = comm.size
    if W == 1:
        return A.view(n0, c1, A.shape[-1])   # the slab is the whole volume: B is A
    send = A.view(c0, W, c1, A.shape[-1]).permute(1, 0, 2, 3).contiguous()
    recv = be.empty_like(send)
    comm.all_to_all(recv, send)
    return recv.view(n0, c1, A.shape[-1])


def _transpose_ba(be, comm, B, n1, c0, c1):
    """B (n0, c1, P) -> A (c0, n1, P): all-to-all #2."""
    W = comm.size
    if W == 1:
        return B.view(c0, n1, B.shape[-1])
    send = B.reshape(W, c0, c1, B.shape[-1])
    recv = be.empty_like(send)
    comm.all_to_all(recv, send)
    return recv.permute(1, 0, 2, 3).reshape(c0, n1, B.shape[-1])


def correct_slab(be, comm: Comm, dims, orig, dec, E, Delta, m: int = 16,
                 max_iters: int = 1000) -> SlabResult:
    """ffcz::correct (pipeline.cpp:26-178) of a volume slab-decomposed along axis 0 (see
    _correct_slab); runs on the backend's stream when it has one."""
    import contextlib
    ctx = be.stream_context() if hasattr(be, "stream_context") else contextlib.nullcontext()
    with ctx:
        return _correct_slab(be, comm, dims, orig, dec, E, Delta, m, max_iters)


def _correct_slab(be, comm: Comm, dims, orig, dec, E, Delta, m: int = 16,
                  max_iters: int = 1000) -> SlabResult:
    """ffcz::correct (pipeline.cpp:26-178) of a volume slab-decomposed along axis 0.

    orig / dec: this rank's (c0, n1, n2) slab (backend tensors, f32 or f64).  Bounds as
    DualBounds holds them (bounds.hpp:11-47), split like the field: E a float or this rank's
    (c0, n1, n2) per-point slab; Delta a float, this rank's (c0, n1, n2) slab of the
    per-component lane (Re == Im, rho mode) or a (Re, Im) pair of such slabs (the full-spectrum
    lanes at this rank's i0 planes).  Array bounds must satisfy DualBounds' invariants (entries
    > 0 and finite, Hermitian-consistent lanes, bounds.cpp:10-59): the caller built them with
    the reference's factories (as FFCZ_BOUNDS_VALIDATED)."""
    import time

    import torch
    n0, n1, n2 = (int(v) for v in dims)
    W, r = comm.size, comm.rank
    timing = os.environ.get("FFCZ_SLAB_TIMING") is not None
    t_last = [time.perf_counter()]

    def _phase(name):  # FFCZ_SLAB_TIMING=1: host time per phase on stderr (synchronises)
        if timing:
            if hasattr(be, "torch") and be.device.type == "cuda":
                be.torch.cuda.synchronize(be.device)
            t = time.perf_counter()
            print(f"[slab r{r}] {name:24s} {1e3 * (t - t_last[0]):9.2f} ms", file=sys.stderr)
            t_last[0] = t
    if len(dims) != 3 or n0 % W or n1 % W:
        raise ValueError("slab decomposition needs a 3-D field with n0, n1 divisible by ranks")
    c0_ = n0 // W
    e_arr = None if np.isscalar(E) else E
    if e_arr is None and not (E > 0.0 and np.isfinite(E)):
        raise be.ValidationError("spatial bound E must be strictly positive and finite")
    if e_arr is not None and tuple(e_arr.shape) != (c0_, n1, n2):
        raise be.ValidationError("per-point bounds must match field size")
    d_lanes = None
    if not np.isscalar(Delta):
        d_lanes = tuple(Delta) if isinstance(Delta, (tuple, list)) else (Delta, None)
        if any(x is not None and tuple(x.shape) != (c0_, n1, n2) for x in d_lanes):
            raise be.ValidationError("per-component bounds must match field size")
    elif not (Delta > 0.0 and np.isfinite(Delta)):
        raise be.ValidationError("frequency bound Delta must be strictly positive and finite")
    if m < 1 or m > 24:
        raise be.ValidationError("shrink_bounds requires 1 <= m <= 24")
    if max_iters < 1:
        raise be.ValidationError("alternating_projection: max_iters must be >= 1")
    if hasattr(be, "set_axes"):
        # one rank: no exchange, so B is the natural layout and the axis the check / clip hooks
        # ride on is free; take the single-volume engine's (the middle axis)
        be.set_axes(W == 1)
    if e_arr is not None or d_lanes is not None:
        # per-component lanes restricted to the half grid on the natural slab (A layout) and
        # moved to the B layout with the same all-to-all as the spectra
        c1_ = n1 // W
        dA = dB = None
        if d_lanes is not None:
            dA = tuple(None if x is None else be.half_lane(x) for x in d_lanes)
            dB = tuple(None if x is None else _transpose_ab(be, comm, x, n0, c0_, c1_).contiguous()
                       for x in dA)
        be.set_bounds(e_arr, dA, dB)
        E = 0.0 if e_arr is not None else E
        Delta = 0.0 if d_lanes is not None else Delta
    else:
        be.set_bounds(None, None, None)
    c0, c1 = n0 // W, n1 // W
    H = n2 // 2 + 1
    N = n0 * n1 * n2
    Ns = c0 * n1 * n2                       # samples of this slab
    base_s = r * Ns                         # global flat index of the slab's first sample
    fw = 1.0 - 2.0 ** -m                    # bounds.cpp:74-85
    slack = 1.0 / (1.0 - 2.0 ** -m) - 1.0 + 2.0 ** -20
    dev = be.device

    # compute_error + preconditions (pipeline.cpp:31-42, projection.cpp:88-94)
    eps = be.zeros_real((c0, n1, n2))
    bad1, bad2 = be.eps0(orig, dec, E, fw, slack, eps)
    big = np.iinfo(np.int64).max
    g1, g2 = comm.min_i64([base_s + bad1 if bad1 >= 0 else big,
                           base_s + bad2 if bad2 >= 0 else big], dev)
    if g1 != big:
        raise be.ValidationError("correct: decompressed data violates the declared spatial "
                                 f"bound at index {g1}")
    if g2 != big:
        raise be.ValidationError("alternating_projection: epsilon0 violates the spatial bound "
                                 f"at index {g2}")

    # ---- alternating projection (projection.cpp:96-126) ----------------------------------
    S = be.zeros_real((c0, n1, n2))
    F_B = be.zeros_half((n0, c1))
    moved_B = be.zeros_moved((n0, c1))
    ls = be.loop_state()
    gate = ls["gate"]
    # fused all-to-all (FFCZ_SLAB_PEER=0 disables): the forward axis-1 pass and the clip +
    # inverse axis-0 pass store straight into the receive buffers of the ranks that own their
    # outputs in the other layout (CUDA IPC / NVLink peer memory), no pack copy, no NCCL buffers
    peer = None
    if (W > 1 and os.environ.get("FFCZ_SLAB_PEER", "1") != "0" and hasattr(be, "peer_ok")
            and be.peer_ok((n0, n1, n2), W)):
        peer = be.peer_setup(comm, (n0, n1, n2))
    if peer is not None:
        A, B = peer["A"], peer["B"]
        be.fwd_local_peer(eps, peer)
        comm.barrier_dev()
    else:
        A = be.zeros_half((c0, n1))
        be.fwd_local(eps, A, N)
        B = None

    # the row step as one fused pass (the single-volume loop's K1) where the backend has it
    fused_row = hasattr(be, "inv_sclip_fwd") and os.environ.get("FFCZ_SLAB_FUSED_ROW", "1") != "0"

    def body_peer(k):
        """body() with the transposes fused into the passes; a device barrier after each
        scattering pass orders it with the receiving ranks' next pass (and their previous pass
        on the same buffer).  Once done, the scattering passes are gated off with the rest, so B
        keeps the last check's spectrum (delta_star)."""
        be.col0_check_dev(B, Delta, fw, ls["red"], gate)
        comm.max_f64_(ls["red"])
        be.decide(ls["red"], ls["state"], gate, max_iters)
        be.col0_clip_inv_peer(Delta, fw, F_B, moved_B, k == 0, peer, gate=gate)
        comm.barrier_dev()
        if fused_row:
            be.inv_sclip_fwd(A, eps, N, E, fw, S, k == 0, gate=gate, col=False)
            be.fwd_local_peer(None, peer, gate=gate)
        else:
            be.inv_local_sclip(A, eps, N, E, fw, S, k == 0, gate=gate)
            be.fwd_local_peer(eps, peer, gate=gate)
        comm.barrier_dev()

    def body(k):
        """One pass of projection.cpp:96-126 with the decision on the device: check, all-reduce
        of (peak, excess), decide (:106-116), clip + inverse, forward.  Every device op returns at
        once when the loop is done; a pass enqueued after that only round-trips the transposes,
        which leaves B (= delta_star) unchanged.  Pass k (from 0) is clip pass k + 1."""
        nonlocal A, B
        B = _transpose_ab(be, comm, A, n0, c0, c1)
        be.col0_check_dev(B, Delta, fw, ls["red"], gate)   # FFT axis 0 + check (in place)
        comm.max_f64_(ls["red"])
        be.decide(ls["red"], ls["state"], gate, max_iters)
        be.col0_clip_inv(B, Delta, fw, F_B, moved_B, k == 0, gate=gate)   # :117-119, axis 0
        A = _transpose_ba(be, comm, B, n1, c0, c1)
        if fused_row:   # axis 1, C2R -> s-clip (:121-124) -> R2C, axis 1 forward
            be.inv_sclip_fwd(A, eps, N, E, fw, S, k == 0, gate=gate)
        else:
            be.inv_local_sclip(A, eps, N, E, fw, S, k == 0, gate=gate)   # axis 1, C2R, :121-124
            be.fwd_local(eps, A, N, gate=gate)

    # one pass queued behind the one being decided: the host waits on an event per pass, never
    # on a value, and the device never idles for the host
    run = body_peer if peer is not None else body
    k = 0
    run(k)
    snaps = [be.snapshot(ls)]
    while True:
        k += 1
        run(k)
        snaps.append(be.snapshot(ls))
        if be.done(snaps.pop(0)):
            break
    passes, converged, residual_f = be.loop_result(ls)
    if peer is not None:
        comm.barrier_dev()      # every rank is past its last (gated) scattering pass
        be.peer_close(peer)
        peer = None
    _phase("loop")
    delta_star = B                                          # FFT(final_eps), pipeline.cpp:114
    # the gate's working set is the peak of the call: drop every loop buffer it does not read
    # (the natural-layout spectrum here, F / the clip map / F_A / freq_cur(A) once consumed)
    A = B = None
    residual_s = comm.max_f64([be.residual_s(eps, E, fw)], dev)[0]

    # ---- FP64 gate (pipeline.cpp:46-176) ---------------------------------------------------
    if passes >= 2:
        # F = mask(delta_star - FFT(eps0 + S)) (the loop marked clipped components only)
        X = be.zeros_real((c0, n1, n2))
        be.eps0_plus_s(orig, dec, S, X)
        A2 = be.zeros_half((c0, n1))
        be.fwd_local(X, A2, N)
        B2 = _transpose_ab(be, comm, A2, n0, c0, c1)
        be.col0_rebuild(B2, delta_star, moved_B, F_B)
        del X, A2, B2
    moved_B = None
    F_A = _transpose_ba(be, comm, F_B, n1, c0, c1)
    F_B = None
    g = be.gate(S, F_A, E, Delta, m, base_h=r * c0 * n1 * H)
    del F_A
    act_s, act_f = comm.sum_i64([g["act_s"], g["act_f"]], dev)
    spat_cur = g["spat_cur"]
    freq_cur_B = _transpose_ab(be, comm, g.pop("freq_cur"), n0, c0, c1)
    esc_s = g["esc_s"]                                     # bool (c0, n1, n2): spatial escapes
    # frequency escapes as global half indices owned (in B) by this rank
    ovf_h = comm.all_gather_rows(g["esc_f_h"].view(-1, 1)).view(-1)
    esc_f_h = be.owned_b(ovf_h, n0, n1, H, r, c1)

    rounds, verified = 0, False
    vs = vf = 0.0
    corrected = be.zeros_real((c0, n1, n2))
    dview = os.environ.get("FFCZ_REPAIR_ORDER") != "reference"
    eps_v = None if dview else be.zeros_real((c0, n1, n2))   # decoder view: only if unverified
    eps_t = be.zeros_real((c0, n1, n2))

    def inverse_to_spatial(fc_B):
        Bw = be.empty_like(fc_B)
        be.col0_plain(fc_B, Bw, +1)
        return _transpose_ba(be, comm, Bw, n1, c0, c1)

    def forward_to_b(x):
        Aw = be.zeros_half((c0, n1))
        be.fwd_local(x, Aw, N)
        Bw = _transpose_ab(be, comm, Aw, n0, c0, c1)
        return Bw

    # decoder-view repair: the round checks the decoder's own view, so a clean
    # round is verify_bounds; FFCZ_REPAIR_ORDER=reference keeps the reference's eps_tilde order
    if converged:
        Aw = Bt = None
        for _ in range(MAX_ESCAPE_ROUNDS):                   # pipeline.cpp:116
            rounds += 1
            Aw = Bt = None                                   # last round's spectra
            Aw = inverse_to_spatial(freq_cur_B)
            dirty_s, vs_r = be.inv_local_repair_verify(Aw, eps_t, N, orig, dec, spat_cur, eps, E,
                                                       esc_s, corrected,
                                                       None if dview else eps_v)
            Aw = None
            Bt = forward_to_b(eps_t)
            viol = be.col0_mark(Bt, Delta)                  # FFT axis 0, |delta~| > Delta
            pos = be.positions(viol)                        # B storage offsets, ascending
            fixed_h = _repair_frequency(be, comm, pos, freq_cur_B, delta_star, Bt,
                                        n0, n1, n2, c1, r)
            esc_f_h = be.merge_sorted(esc_f_h, fixed_h)
            dirty = comm.sum_i64([int(dirty_s) + int(pos.numel() > 0)], dev)[0]
            if dirty == 0:                                  # :161, clean round
                vs = comm.max_f64([vs_r], dev)[0]
                if dview:
                    vf = 0.0    # the round's own forward transform was of the decoder view
                else:
                    Bv = forward_to_b(eps_v)
                    vf = comm.max_f64([be.col0_verify(Bv, Delta)], dev)[0]
                verified = True
                break
    if not verified:
        # apply_edits + verify_bounds on the decoder view (archive.cpp:262-297)
        if eps_v is None:
            eps_v = eps_t                                    # the rounds' scratch is free now
        Aw = inverse_to_spatial(freq_cur_B)
        vs_r = be.inv_local_verify(Aw, eps_v, N, orig, dec, spat_cur, E, corrected)
        vs = comm.max_f64([vs_r], dev)[0]
        Bv = forward_to_b(eps_v)
        vf = comm.max_f64([be.col0_verify(Bv, Delta)], dev)[0]

    _phase("gate + repair rounds")
    # escapes in std::map order: spatial by index, then frequency by half index
    sp_idx = be.nonzero_flat(esc_s)
    sp = torch.stack([sp_idx.double() + base_s, be.take_real(spat_cur, sp_idx)], 1) \
        if sp_idx.numel() else torch.zeros((0, 2), dtype=torch.float64, device=dev)
    fr_vals = be.values_at_h(freq_cur_B, esc_f_h, n1, H, r, c1)
    fr = torch.stack([esc_f_h.double(), fr_vals.real, fr_vals.imag], 1) \
        if esc_f_h.numel() else torch.zeros((0, 3), dtype=torch.float64, device=dev)
    sp_all = comm.all_gather_rows(sp).cpu().numpy()
    fr_all = comm.all_gather_rows(fr).cpu().numpy()
    fr_all = fr_all[np.argsort(fr_all[:, 0], kind="stable")]
    escapes = EscapeList(sp_all, fr_all)
    _phase("escape lists")
    return SlabResult(
        iterations=max(passes, 1), converged=converged, residual_f=residual_f,
        residual_s=residual_s, active_spatial=int(act_s), active_frequency=int(act_f),
        verify_ok=(vs == 0.0 and vf == 0.0), verify_max_spatial_excess=vs,
        verify_max_freq_excess=vf, escape_rounds=rounds,
        spatial_flags=g["keep_s"], frequency_flags=g["keep_f"], spatial_codes=g["codes_s"],
        frequency_codes=g["codes_f"], escapes=escapes, corrected=corrected)


def _repair_frequency(be, comm, pos, freq_cur_B, delta_star, delta_tilde, n0, n1, n2, c1, r):
    """Frequency side of one escape-repair round (pipeline.cpp:140-153) on the B layout.

    Violating components are pinned to freq_cur + (delta_star - delta_tilde) (values of this
    round's freq_cur).  Components on the k2 = 0 / n2/2 planes also set their conjugate partner
    (-i0, -i1, k2); the reference visits half indices in ascending order, so when both partners
    violate the larger index's repair wins.  Partners may be owned by another rank: the plane
    repairs are all-gathered (they are few).  Returns the sorted global half indices this rank
    repaired (escape set additions it owns)."""
    import torch
    H = n2 // 2 + 1
    P = freq_cur_B.shape[-1]
    i0 = torch.div(pos, c1 * P, rounding_mode="floor")
    rem = pos - i0 * c1 * P
    i1 = torch.div(rem, P, rounding_mode="floor") + r * c1
    k2 = rem % P
    h = (i0 * n1 + i1) * H + k2
    flat_cur = freq_cur_B.view(-1)
    rv = flat_cur[pos] + (delta_star.view(-1)[pos] - delta_tilde.view(-1)[pos])
    plane = (k2 == 0) | (2 * k2 == n2)
    mi0 = (n0 - i0) % n0
    mi1 = (n1 - i1) % n1
    hm = (mi0 * n1 + mi1) * H + k2
    self_pair = plane & (hm == h)
    # off-plane (and self-conjugate) components: local
    loc = ~plane | self_pair
    flat_cur[pos[loc]] = rv[loc]
    fixed = [h[loc]]
    # plane pairs: every rank sees every plane violation (h, re, im)
    pl = ~loc
    rows = torch.stack([h[pl].double(), rv[pl].real, rv[pl].imag], 1) if int(pl.sum()) else \
        torch.zeros((0, 3), dtype=torch.float64, device=pos.device)
    allp = comm.all_gather_rows(rows)
    if allp.shape[0]:
        ph = allp[:, 0].long()
        pv = torch.complex(allp[:, 1], allp[:, 2])
        pk2 = ph % H
        prow = torch.div(ph, H, rounding_mode="floor")
        pi0 = torch.div(prow, n1, rounding_mode="floor")
        pi1 = prow % n1
        pm = (((n0 - pi0) % n0) * n1 + (n1 - pi1) % n1) * H + pk2
        viol_set = set(ph.tolist())
        # winner per pair: the larger violating index (ascending visit order)
        targets_h, targets_v = [], []
        for a, b, v in zip(ph.tolist(), pm.tolist(), pv.tolist()):
            if b in viol_set and b > a:
                continue                     # the partner (larger) repair wins
            targets_h += [a, b]
            targets_v += [v, np.conj(v)]
        th = torch.tensor(targets_h, dtype=torch.int64, device=pos.device)
        tv = torch.tensor(targets_v, dtype=torch.complex128, device=pos.device)
        # keep those owned (in B) by this rank
        trow = torch.div(th, H, rounding_mode="floor")
        ti0 = torch.div(trow, n1, rounding_mode="floor")
        ti1 = trow % n1
        tk2 = th % H
        own = torch.div(ti1, c1, rounding_mode="floor") == r
        off = (ti0 * c1 + (ti1 - r * c1)) * P + tk2
        flat_cur[off[own]] = tv[own].to(flat_cur.dtype)
        fixed.append(th[own])
    out = torch.cat(fixed) if fixed else torch.zeros(0, dtype=torch.int64, device=pos.device)
    return torch.unique(out)
