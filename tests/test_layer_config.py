"""Layer-config validation on the host (no GPU): the DECOUPLED group size is
resolved and checked at create exactly as the reference's run_dispatch
precheck (protocols.cpp:348-359) and assign_groups (:77-88) do — a size that
does not divide every PE's remote tile count is a ConfigError, never a device
plan error that leaves peers spinning."""
import pytest

import paper_2605_00686_b200 as pb

QWEN3 = pb.ModelConfig("qwen3", 2048, 768, 128, 8)


def test_fixed_group_size_must_divide_every_pe_tile_count():
    # Qwen3 EP=4, S=4096: 2 tiles per (src, expert), 32 experts per destination
    # -> 192 remote tiles per PE (both directions)
    assert pb.resolve_group_size(QWEN3, 4096, 4, protocol=pb.combined_protocol(16)) == 16
    with pytest.raises(pb.ConfigError, match="does not divide"):
        pb.resolve_group_size(QWEN3, 4096, 4, protocol=pb.combined_protocol(5))
    # Zipf counts: known on the host for every PE from the reference's seeded draws
    with pytest.raises(pb.ConfigError, match="does not divide"):
        pb.resolve_group_size(QWEN3, 4096, 4, routing="zipf", skew=1.2, protocol=pb.combined_protocol(7))
    with pytest.raises(pb.ConfigError, match="does not divide"):
        pb.MoELayer(QWEN3, 4096, rank=0, world=4, routing="balanced", protocol=pb.combined_protocol(5))


def test_group_size_needs_reference_routing():
    with pytest.raises(pb.ConfigError, match="reference routing"):
        pb.resolve_group_size(QWEN3, 4096, 2, routing="gate", protocol=pb.combined_protocol(8))
    assert pb.resolve_group_size(QWEN3, 4096, 2, routing="gate", protocol=pb.combined_protocol(0)) == 0


@pytest.mark.parametrize("P,S,want", [(2, 4096, 32), (4, 4096, 16), (8, 4096, 8), (4, 1024, 8), (8, 1024, 8),
                                      (2, 256, 16)])
def test_auto_group_size(P, S, want):
    """GROUP_AUTO: the largest common divisor g of the PEs' remote tile counts
    with 8 <= g <= tiles-per-destination / 4, else per destination (0)."""
    g = pb.resolve_group_size(QWEN3, S, P, protocol=pb.combined_protocol(-1))
    assert g == want
    if g:
        tiles_per_dst = -(-(S * 8 // 128) // 128) * (128 // P)
        assert tiles_per_dst % g == 0 and g >= 8
        assert tiles_per_dst // g >= 4 or tiles_per_dst < 32


def test_per_tile_protocols_report_group_size_one():
    assert pb.resolve_group_size(QWEN3, 4096, 4, protocol=pb.vanilla_protocol()) == 0


def test_pdl_off_when_ranks_share_a_device(monkeypatch):
    """MoELayer(pdl=None): PERSEUS_F_NO_PDL is set when the EP world is larger than
    the visible device count (several ranks per GPU: a grid waiting for its PDL
    primary holds up the work distributor) or PERSEUS_SHARED_DEVICE=1, never for
    one process per GPU; pdl=True / False override.  The create call is
    intercepted, so no GPU is needed."""
    import torch
    from paper_2605_00686_b200 import _lib, layer as layer_mod
    seen = []

    class FakeLib:
        def __getattr__(self, name):
            return getattr(_lib.lib, name)

        @staticmethod
        def perseus_layer_create(cfg, rank, world, device, h):
            seen.append(cfg._obj.flags)
            return 0

    monkeypatch.setattr(layer_mod, "lib", FakeLib())
    monkeypatch.setattr(torch.cuda, "device_count", lambda: 4)
    monkeypatch.delenv("PERSEUS_SHARED_DEVICE", raising=False)

    def flags_for(world, **kw):
        seen.clear()
        layer_mod.MoELayer(QWEN3, 1024, rank=0, world=world, **kw)
        return seen[-1]

    assert not flags_for(4) & _lib.F_NO_PDL          # one process per GPU
    assert flags_for(8) & _lib.F_NO_PDL              # 8 ranks on 4 GPUs
    assert not flags_for(8, pdl=True) & _lib.F_NO_PDL
    assert flags_for(2, pdl=False) & _lib.F_NO_PDL
    monkeypatch.setenv("PERSEUS_SHARED_DEVICE", "1")
    assert flags_for(2) & _lib.F_NO_PDL
