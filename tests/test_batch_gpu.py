"""NEXT-4 batch coalescing on the GPU (K6) against oracle O12, bit-exact."""
import numpy as np
import pytest

from nalar_gen import AFF_NONE, c2, c4, random_table
from oracle import oracle_epoch

pytestmark = pytest.mark.gpu


def _nalar():
    from paper_2601_05109_b200 import nalar
    return nalar


def check(s, mb, policy="srtf", epochs=3, flags=0):
    nalar = _nalar()
    o = oracle_epoch(s, policy, batch={"t_max_batch": mb, "f_method": s.f_method})
    ctx = nalar.Context.for_snapshot(s, flags=flags)
    ctx.set_policy_params(t_max_batch=mb, n_types=s.n_types)
    ctx.upload(s)
    for _ in range(epochs):
        ctx.epoch(policy)
        g = ctx.fetch()
        assert np.array_equal(g["batch_head"], o["batch_head"]), np.nonzero(g["batch_head"] != o["batch_head"])
        assert g["n_batches"] == o["n_batches"]
        assert np.array_equal(g["assign_row"], o["assign_row"])
    ctx.close()
    return o


@pytest.mark.parametrize("seed", range(60))
def test_batch_random(seed):
    rng = np.random.default_rng(seed)
    s = random_table(seed, n_workflows=3 + seed % 8, max_rows=4 + seed % 25, n_types=1 + seed % 3,
                     inst_per_type=(1, 3), consistent=seed % 2 == 0, max_cap=2 + seed % 9, p_pin=0.3)
    s.t_affinity[:] = AFF_NONE
    s.f_method = rng.integers(0, 1 + seed % 4, s.n_futures)
    check(s, rng.integers(0, 5, s.n_types), ["fcfs", "srtf", "lpt"][seed % 3])


@pytest.mark.parametrize("mk", [lambda: c2(1), c4])
def test_batch_full_size(mk):
    s = mk()
    rng = np.random.default_rng(3)
    s.f_method = rng.integers(0, 3, s.n_futures)
    mb = np.where(s.t_affinity == AFF_NONE, 4, 0)
    o = check(s, mb)
    assert o["n_batches"] > 0


def test_batch_managed_state_rejected_and_off():
    nalar = _nalar()
    s = c4()
    ctx = nalar.Context.for_snapshot(s)
    ctx.upload(s)
    ctx.set_policy_params(t_max_batch=np.full(8, 4), n_types=8)      # SESSION / STATEFUL types too
    with pytest.raises(nalar.NalarError):
        ctx.epoch("srtf")
    ctx.set_policy_params()
    ctx.epoch("srtf")
    g = ctx.fetch()
    assert g["n_batches"] == 0 and (g["batch_head"] == -1).all()
    ctx.close()


@pytest.mark.parametrize("unpin", [False, True])
def test_batch_long_sequences_fallback(unpin):
    """Instances receiving more futures than K6 stages in shared memory (1024
    per sequence): one instance per type takes all of its type's work, so its
    sequence (phase B, or phase A once every future is pinned to it) exceeds
    the staging and the global-memory merge runs -- the same batches."""
    from nalar_gen import swe_table
    s = swe_table(400000, seed=7)
    s.t_affinity[:] = AFF_NONE
    first = np.array([np.nonzero(s.i_type == t)[0][0] for t in range(s.n_types)])
    cap = np.zeros(s.n_instances, dtype=s.i_cap.dtype)
    cap[first] = 1000000
    s.i_cap[:] = cap
    s.i_base_load[:] = 0
    if unpin:
        s.f_pin[:] = np.where(s.f_state == 0, first[s.f_type], s.f_pin)
    rng = np.random.default_rng(5)
    s.f_method = rng.integers(0, 3, s.n_futures)
    o = check(s, np.full(s.n_types, 5), epochs=2)
    inst = o["instance"][o["status"] == 7]
    assert np.bincount(inst).max() > 1024
