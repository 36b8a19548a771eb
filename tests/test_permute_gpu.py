"""a7: permute materialisation on the GPU, bit-exact against the reference / oracle."""
import itertools

import numpy as np
import pytest

import tnkit_np as oracle
from tnb_testutil import load

import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import storage

pytestmark = pytest.mark.gpu


def test_golden_permute_cases(cuda):
    z, meta = load("permute.npz")
    for k, c in enumerate(meta["cases"]):
        t = storage.DenseTensor(z[f"in{k}"])
        p = t.permute(*c["perm"])
        assert p.same_data(t)  # lazy
        got = p.contiguous()
        assert got.is_contiguous and got.shape == tuple(z[f"out{k}"].shape)
        assert np.array_equal(got.numpy(), z[f"out{k}"]), c


def test_acceptance_storage_reordering(cuda):
    t = storage.arange(8).reshape(2, 2, 2).permute(0, 2, 1)
    assert list(t.storage().cpu().numpy()) == [0, 1, 2, 3, 4, 5, 6, 7]
    t.contiguous_()
    assert list(t.storage().cpu().numpy()) == [0, 2, 1, 3, 4, 6, 5, 7]


def test_contiguous_of_contiguous_shares_and_reshape(cuda):
    t = storage.arange(24).reshape(2, 3, 4)
    assert t.contiguous().same_data(t) and t.reshape(6, 4).same_data(t)
    p = t.permute(2, 0, 1)
    r = p.reshape(4, 6)
    assert not r.same_data(t)
    assert np.array_equal(r.numpy(), np.arange(24.0).reshape(2, 3, 4).transpose(2, 0, 1).reshape(4, 6))
    with pytest.raises(ValueError):
        t.permute(0, 0, 1)


@pytest.mark.parametrize("dtype", [np.float64, np.complex128])
def test_all_rank4_perms_bitexact(cuda, dtype):
    src = oracle.uniform([12, 7, 16, 9], dtype=dtype, seed=3)
    t = storage.DenseTensor(src)
    for perm in itertools.permutations(range(4)):
        assert np.array_equal(t.permute(*perm).contiguous().numpy(), oracle.permute_contiguous(src, perm)), perm


@pytest.mark.parametrize("dtype", [np.float64, np.complex128, np.int64, np.bool_])
def test_random_rank6_and_odd_shapes(cuda, dtype):
    rng = np.random.default_rng(11)
    for shape in [(16,) * 6, (3, 5, 7, 2, 9, 4), (1, 17, 1, 33, 2, 1), (65, 3, 129)]:
        src = (rng.random(shape) * 100).astype(dtype) if dtype != np.bool_ else rng.random(shape) < 0.5
        if dtype == np.complex128:
            src = src + 1j * rng.random(shape)
        t = storage.DenseTensor(src)
        for _ in range(4):
            perm = tuple(int(x) for x in rng.permutation(len(shape)))
            assert np.array_equal(t.permute(*perm).contiguous().numpy(), oracle.permute_contiguous(src, perm))


def test_chained_lazy_permutes(cuda):
    src = oracle.uniform([4, 5, 6, 7], seed=9)
    t = storage.DenseTensor(src).permute(3, 1, 0, 2).permute(1, 3, 0, 2)
    want = src.transpose(3, 1, 0, 2).transpose(1, 3, 0, 2)
    assert np.array_equal(t.contiguous().numpy(), np.ascontiguousarray(want))


@pytest.mark.parametrize("shape", [(64, 64, 64, 64), (16,) * 6])
def test_full_size_bench_shapes_checksum(cuda, shape):
    """BASELINE config C2 sizes: checksum properties (sum preserved, spot values)."""
    import torch
    src = oracle.uniform(list(shape), seed=21)
    t = storage.DenseTensor(src)
    rng = np.random.default_rng(1)
    for _ in range(3):
        perm = tuple(int(x) for x in rng.permutation(len(shape)))
        out = t.permute(*perm).contiguous()
        dev = out.storage()
        assert float(dev.sum()) == pytest.approx(float(src.sum()), rel=1e-12)
        idx = [tuple(int(rng.integers(0, d)) for d in out.shape) for _ in range(50)]
        host = out.numpy()
        for i in idx:
            assert host[i] == src[tuple(i[perm.index(a)] for a in range(len(shape)))]
        assert np.array_equal(host, oracle.permute_contiguous(src, perm))


@pytest.mark.parametrize("seed", range(6))
def test_random_ranks_dims_dtypes_bitexact(cuda, seed):
    """Fuzz over every planner path (row gathers, TMA bulk rows, t2d tiles, general tiles):
    ranks 1-16 (TNB_MAX_RANK), random extents (unit axes included), four dtypes, random
    permutations -- bit-exact against the oracle's np.ascontiguousarray(view)."""
    rng = np.random.default_rng(500 + seed)
    for _ in range(12):
        rank = int(rng.integers(1, 17))
        choices = [1, 2, 3, 5, 8, 16, 17, 31, 64, 100] if rank <= 8 else [1, 2, 3]
        while True:
            shape = tuple(int(rng.choice(choices)) for _ in range(rank))
            if int(np.prod(shape)) <= (1 << 21):
                break
        dtype = [np.float64, np.complex128, np.int64, np.bool_][int(rng.integers(0, 4))]
        if dtype == np.bool_:
            src = rng.random(shape) < 0.5
        elif dtype == np.int64:
            src = rng.integers(-1000, 1000, size=shape)
        else:
            src = rng.standard_normal(shape).astype(dtype)
            if dtype == np.complex128:
                src = src + 1j * rng.standard_normal(shape)
        t = storage.DenseTensor(src)
        perm = tuple(int(x) for x in rng.permutation(rank))
        assert np.array_equal(t.permute(*perm).contiguous().numpy(), oracle.permute_contiguous(src, perm)), \
            (shape, perm, dtype)


def test_generic_tiled_path_bit_exact(cuda):
    """Permutes that the transpose / row kernels do not take (1-byte bools, int64 / float64
    with inner axes shorter than 64 bytes, a partial input axis that is also inner on the
    output side) go through the generic tiled kernel: bit-exact against numpy."""
    rng = np.random.default_rng(17)
    cases = [((16,) * 6, np.bool_), ((64, 64, 64), np.bool_), ((50, 40, 6, 3), np.float64),
             ((300, 5, 7, 4), np.int64), ((16, 16, 16, 16, 16, 16), np.float64), ((33, 7, 65, 3, 5), np.complex128)]
    for shape, dt in cases:
        if dt == np.bool_:
            src = rng.integers(0, 2, size=shape).astype(np.bool_)
        elif dt == np.int64:
            src = rng.integers(-1000, 1000, size=shape).astype(np.int64)
        elif dt == np.complex128:
            src = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(dt)
        else:
            src = rng.standard_normal(shape).astype(dt)
        t = storage.DenseTensor(src)
        for _ in range(4):
            p = tuple(int(x) for x in rng.permutation(len(shape)))
            got = t.permute(*p).contiguous().numpy()
            assert np.array_equal(got, np.ascontiguousarray(src.transpose(p))), (shape, dt, p)
