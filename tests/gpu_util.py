"""Shared helpers of the GPU parity tests (test infrastructure)."""
import numpy as np

from oracle.oracle import LayerShape


def bf16_bits(t):
    """torch bf16 tensor -> numpy uint16 bits (host)."""
    import torch
    return t.detach().view(torch.int16).cpu().numpy().view(np.uint16)


def run_emulated(pb, model, S, P, routing="balanced", skew=0.0, seed=1, protocol=None, reps=1, before=None):
    """P EP ranks emulated on ONE device: phase p of every rank completes
    before phase p+1 of any rank (no cross-launch spin-waits on one GPU)."""
    import torch
    layers = [pb.MoELayer(model, S, rank=r, world=P, device=0, routing=routing, skew=skew, seed=seed,
                          protocol=protocol) for r in range(P)]
    if P > 1:
        pb.MoELayer.connect_local(layers)
    if before is not None:
        before(layers)
    xs = [torch.empty(S, model.hidden_dim, dtype=torch.bfloat16, device="cuda") for _ in range(P)]
    outs = [torch.zeros_like(x) for x in xs]
    for r, l in enumerate(layers):
        l.fill_synthetic_x(xs[r], seed)
    for _ in range(reps):
        for phase in (0, 1, 2, 3):
            for r, l in enumerate(layers):
                l.forward_phase(phase, xs[r], outs[r])
    torch.cuda.synchronize()
    return layers, xs, outs


def shape_of(model, S, P):
    return LayerShape(model.hidden_dim, model.intermediate_dim, model.experts, model.top_k, S, P)


def assert_close(out_f32, ref_f32, tol=1e-2, what=""):
    """bf16 tolerance of north_star: max-abs error relative to max |ref| and
    the normwise relative error both <= tol (1e-2)."""
    err = np.abs(out_f32 - ref_f32)
    scale = np.abs(ref_f32).max()
    rel_max = err.max() / scale
    rel_norm = np.linalg.norm(out_f32 - ref_f32) / np.linalg.norm(ref_f32)
    assert np.all(np.isfinite(out_f32)), f"{what}: non-finite output"
    assert rel_max <= tol and rel_norm <= tol, f"{what}: rel_max={rel_max:.3e} rel_norm={rel_norm:.3e}"
    return rel_max, rel_norm


def run_concurrent(pb, model, S, P, routing="balanced", skew=0.0, seed=1, protocol=None, reps=1, before=None,
                   sync_each=True, pair=True, flags=0):
    """P EP ranks on ONE device running the PRODUCTION path concurrently: every
    rank's full forward (route -> permute + plan -> fused persistent k_moe2 on
    CTA pairs -> combine) on its own stream, ranks synchronising only through
    device flag words in each other's symmetric buffers — the same kernels and
    signalling as one process per GPU, with each rank's persistent grid capped
    to 1/P of the SMs (PERSEUS_NUM_SMS, read at create) so all P fused kernels
    are co-resident, and launched without PDL (PERSEUS_F_NO_PDL): measured on
    B200, a rank's grid waiting for its programmatic-dependent-launch primary
    holds up the work distributor, so another rank's fused kernel that the
    primary waits for was left unscheduled until the waits timed out (always
    at P >= 3, sometimes at P = 2); one process per GPU never shares a device.
    """
    import os
    import torch
    n_sms = torch.cuda.get_device_properties(0).multi_processor_count
    old = os.environ.get("PERSEUS_NUM_SMS")
    os.environ["PERSEUS_NUM_SMS"] = str((n_sms // P) & ~1)
    try:
        layers = [pb.MoELayer(model, S, rank=r, world=P, device=0, routing=routing, skew=skew, seed=seed,
                              protocol=protocol, pair=pair, pdl=False, flags=flags) for r in range(P)]
    finally:
        if old is None:
            os.environ.pop("PERSEUS_NUM_SMS", None)
        else:
            os.environ["PERSEUS_NUM_SMS"] = old
    if P > 1:
        pb.MoELayer.connect_local(layers)
    if before is not None:
        before(layers)
    xs = [torch.empty(S, model.hidden_dim, dtype=torch.bfloat16, device="cuda") for _ in range(P)]
    outs = [torch.zeros_like(x) for x in xs]
    for r, l in enumerate(layers):
        l.fill_synthetic_x(xs[r], seed)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(P)]
    for _ in range(reps):
        for r, l in enumerate(layers):
            l.forward(xs[r], outs[r], stream=streams[r])
        if sync_each:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    return layers, xs, outs
