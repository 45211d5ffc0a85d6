"""CPU checks of the slab layout (which levels are distributed, level scales)."""

import pytest

from paper_2405_19991_b200.slab import SlabLayout, level_scales


def test_slab_layout_levels():
    # every splittable level distributed (min_local 0): 32, 16, 8, 4, 2 planes per rank
    L = SlabLayout.make((256, 256, 256), 8, min_local=0)
    assert L.chain[0] == (256, 256, 256) and L.nlev_dist == 5 and L.chain[5] == (8, 8, 8)
    assert L.scales[2] == (1 / 16, 1 / 16, 1 / 16)
    assert level_scales([(8, 8, 8), (4, 4, 4)])[1] == (0.25, 0.25, 0.25)
    L1 = SlabLayout.make((32, 32, 32), 1, min_local=0)
    assert L1.nlev_dist == 3 and L1.chain[3] == (4, 4, 4)
    # default: a level stays on slabs while each rank keeps >= 65536 vertices
    assert SlabLayout.make((256, 256, 256), 8).chain[SlabLayout.make((256, 256, 256), 8).nlev_dist] == (64, 64, 64)
    assert SlabLayout.make((256, 256, 256), 1).nlev_dist == 3          # 256, 128, 64 on slabs; 32^3 agglomerated
    assert SlabLayout.make((512, 512, 512), 8).nlev_dist == 3          # 128^3 / 8 = 262144 >= 65536; 64^3 agglomerated
    assert SlabLayout.make((16, 8, 8), 2).nlev_dist == 1               # level 0 is always distributed
    with pytest.raises(ValueError):
        SlabLayout.make((6, 8, 8), 4)
