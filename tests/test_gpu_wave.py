"""GPU: the fused wavefront half-steps (wave.cu: K-Q + K-Cb and K-M2 + K-CTe in
one persistent kernel each; SFEEC_WAVE=1, off by default because measured
slower) are bitwise the unfused 4-kernel chain, for every item size / lag /
ticket batch of the plan and with or without CUDA-graph replay."""
import numpy as np
import pytest

import paper_2301_01753_b200 as S
from paper_2301_01753_b200 import configs
from tests.test_gpu_delta import layout_env

pytestmark = pytest.mark.gpu


def _state(s, seed):
    rng = np.random.default_rng(seed)
    return S.make_state(S.Formulation.BE, rng.standard_normal(s._n2), rng.standard_normal(s._n1))


def _run(make, steps, seed, **env):
    with layout_env(**env):
        s = make()
        out = s.advance(_state(s, seed), steps)
        return out, s.fused(), s.last_launches()


def _assert_same(a, b):
    assert np.array_equal(a.first, b.first) and np.array_equal(a.e, b.e)


@pytest.mark.parametrize("n", [6, 16])
@pytest.mark.parametrize("steps", [1, 7, 40])  # 40: the CUDA-graph replay of 32 pairs
def test_tet_wave_bitwise_equals_unfused(n, steps):
    make = lambda: S.tet_device_scheme(n, 0.1, 3, dt=0.01)
    ref, f0, l0 = _run(make, steps, n, SFEEC_WAVE=0)
    out, f1, l1 = _run(make, steps, n, SFEEC_WAVE=1)
    assert f0 == 0 and f1 & 2 and (n < 16 or f1 == 3)  # small meshes keep Q in CSR
    if f1 == 3:
        assert l1 == l0 // 2  # two launches per step instead of four
    _assert_same(out, ref)


@pytest.mark.parametrize("entries,lag,batch", [(1, 0, 1), (64, 3, 5), (100000, 0, 2),
                                               (8192, 10**9, 16)])
def test_tet_wave_plan_shapes(entries, lag, batch):
    """Tiny items (many flags), no lag (consumers right behind their
    producers), huge items and an infinite lag (all consumers at the end)."""
    make = lambda: S.tet_device_scheme(16, 0.15, 5, dt=0.01)
    ref, _, _ = _run(make, 12, 1, SFEEC_WAVE=0)
    out, f, _ = _run(make, 12, 1, SFEEC_WAVE=1, SFEEC_WAVE_ENTRIES=entries, SFEEC_WAVE_LAG=lag,
                     SFEEC_WAVE_BATCH=batch)
    assert f == 3, f
    _assert_same(out, ref)


def test_host_built_tet_scheme_wave():
    sys_ = configs.tet_system(7, 0.1, 2)
    make = lambda: S.SplitScheme(S.SplitKind.Strang, 0.01, sys_.q, sys_.c, sys_.m2, div=sys_.d,
                                 warn_cfl=False)
    ref, _, _ = _run(make, 35, 4, SFEEC_WAVE=0)
    out, f, _ = _run(make, 35, 4, SFEEC_WAVE=1)
    assert f & 2, f
    _assert_same(out, ref)


def test_cubical_lattice_wave():
    """Lumped masses: Q and M2 are uniform-valued (signed-layout) width-1
    operators, which the wavefront kernel does not take: the chain stays
    unfused and unchanged."""
    c, d = S.yee_operators(6, 5, 7, 1.0, 0.8, 1.25, bc=1)
    dv = 1.0 * 0.8 * 1.25
    q, m2 = S.scaled_identity(c.cols, 1.0 / dv), S.scaled_identity(c.rows, dv)
    make = lambda: S.SplitScheme(S.SplitKind.Strang, 0.2, q, c, m2, div=d, warn_cfl=False)
    ref, _, _ = _run(make, 20, 5, SFEEC_WAVE=0)
    out, f, _ = _run(make, 20, 5, SFEEC_WAVE=1)
    _assert_same(out, ref)
    assert f == 0


def test_p2_wave():
    make = lambda: S.p2_device_scheme(3, 0.1, 2, dt=0.005)
    ref, _, _ = _run(make, 9, 6, SFEEC_WAVE=0)
    out, f, _ = _run(make, 9, 6, SFEEC_WAVE=1)
    _assert_same(out, ref)


def test_wave_is_off_by_default():
    import os
    assert "SFEEC_WAVE" not in os.environ
    s = S.tet_device_scheme(16, 0.1, 3, dt=0.01)
    s.advance(_state(s, 1), 2)
    assert s.fused() == 0


def test_lie_trotter_wave():
    sys_ = configs.tet_system(4, 0.1, 2)
    lt = S.SplitScheme(S.SplitKind.LieTrotter, 0.01, sys_.q, sys_.c, sys_.m2, warn_cfl=False)
    ref = S.SplitScheme(S.SplitKind.LieTrotter, 0.01, sys_.q, sys_.c, sys_.m2, warn_cfl=False)
    st = _state(lt, 3)
    with layout_env(SFEEC_WAVE=0):
        x = ref.advance(st, 5)
    with layout_env(SFEEC_WAVE=1):
        y = lt.advance(st, 5)  # Lie-Trotter: He and Ha fused one by one
    _assert_same(x, y)
