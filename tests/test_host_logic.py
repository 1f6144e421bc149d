"""Host-side launch-mapping logic (no GPU needed): every mapping the
package picks for the hyperplane ILU0 kernel is one the kernel accepts
(include/ntdgpu.h ntd_ilu0_hp_apply_ex limits), across grids and batch sizes."""

import pytest

from paper_1909_09771_b200 import device as D


GRIDS = [(32, 32, 32), (64, 64, 64), (96, 96, 96), (128, 128, 128), (350, 350, 350), (21, 37, 10),
         (7, 5, 9), (200, 40, 64), (12, 600, 20), (1, 1, 8)]


@pytest.mark.parametrize("grid", GRIDS, ids=[f"{g[0]}x{g[1]}x{g[2]}" for g in GRIDS])
def test_hp_mappings_within_kernel_limits(grid):
    nx, ny, nz = grid
    n = nx * ny * nz
    for split in (n // 2, (nz // 2) * nx * ny):
        for systems in (1, 2, 4, 8, 16, 32, 64):
            cfg = D.ilu0_hp_config(nx, ny, nz, split, systems)
            if cfg is None:
                continue
            nc, w = cfg[:2]
            links = cfg[2] if len(cfg) > 2 else 0
            g = (ny + 31) // 32
            nxy = nx * ny
            assert split % nxy == 0
            nk = max(split // nxy, nz - split // nxy)
            umax = -(-nk // nc) * g
            upw = -(-umax // w)
            assert 1 <= nc <= nk and umax <= 380 and 1 <= upw <= 8
            assert w <= (24 if upw == 1 else 16)
            if nc > 16:  # global-memory links, cooperative launch: a lone system, one CTA per SM
                assert systems == 1 and 2 * systems * nc <= 148
            elif links == 2:  # global-memory links inside a cluster launch
                assert systems <= 8
            else:
                assert links in (0, 1)
    assert D.ilu0_hp_config(96, 96, 96, 96 ** 3 // 2, 64) is None  # the batch keeps the skewed kernel
    assert D.ilu0_hp_config(350, 350, 350, 350 ** 3 // 2, 1)[0] > 16
