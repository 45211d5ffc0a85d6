"""CPU checks of the slab layout (which levels are distributed, level scales)."""

import pytest

from paper_2405_19991_b200.slab import SlabLayout, level_scales


def test_slab_layout_levels():
    L = SlabLayout.make((256, 256, 256), 8)
    # 32, 16, 8, 4, 2 planes per rank on levels 0-4; 8^3 agglomerated
    assert L.chain[0] == (256, 256, 256) and L.nlev_dist == 5 and L.chain[5] == (8, 8, 8)
    assert L.scales[2] == (1 / 16, 1 / 16, 1 / 16)
    assert level_scales([(8, 8, 8), (4, 4, 4)])[1] == (0.25, 0.25, 0.25)
    L1 = SlabLayout.make((32, 32, 32), 1)
    assert L1.nlev_dist == 3 and L1.chain[3] == (4, 4, 4)
    with pytest.raises(ValueError):
        SlabLayout.make((6, 8, 8), 4)
