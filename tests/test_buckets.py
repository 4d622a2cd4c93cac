"""CPU: gradient-bucket fusion bookkeeping through the C-ABI (host-only
container: no gradients attached) against the reference's own assertions for
GradBucket / make_gradient_buckets (test_collectives.cpp:174-233)."""
import pytest

from paper_2205_10034_b200.moesim import GradBuckets


def sm64(seed):
    """rng.hpp SplitMix64 stream (test_collectives.cpp:196 uses SplitMix64(23))."""
    s = seed & (2**64 - 1)
    while True:
        s = (s + 0x9E3779B97F4A7C15) & (2**64 - 1)
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        yield z ^ (z >> 31)


def single(ids):
    """One GradBucket(ids): capacity = len(ids); registration order == ids."""
    b = GradBuckets(list(reversed(ids)), len(ids))
    assert len(b) == 1 and b.ids(0) == list(ids)
    return b


def test_capacity_one_flushes_on_every_push():
    b = single([42])
    assert b.push(42) == 0 and b.ids(0) == [42]


def test_out_of_order_arrivals_keep_registration_order():
    b = single([1, 2, 3])
    assert b.push(3) is None
    assert b.push(1) is None
    assert b.push(2) == 0
    assert b.ids(0) == [1, 2, 3]


def test_duplicate_and_foreign_pushes_are_errors():
    b = single([1, 2])
    assert b.push(1) is None
    with pytest.raises(ValueError, match="duplicate push of gradient 1"):
        b.push(1)
    with pytest.raises(ValueError, match="gradient 99 is not registered"):
        b.push(99)


def test_random_arrival_orders_never_double_flush():
    rng = sm64(23)
    for _ in range(30):
        n = 1 + next(rng) % 8
        ids = list(range(100, 100 + n))
        arrival = list(ids)
        for i in range(n, 1, -1):
            j = next(rng) % i
            arrival[i - 1], arrival[j] = arrival[j], arrival[i - 1]
        b = single(ids)
        flushes = 0
        for i, a in enumerate(arrival):
            r = b.push(a)
            if r is not None:
                flushes += 1
                assert i == n - 1 and b.ids(r) == ids
        assert flushes == 1
        b.reset()
        assert (b.push(ids[0]) is None) == (n > 1)


def test_partitioning_registers_in_reverse_layer_order():
    b = GradBuckets([1, 2, 3, 4, 5], 2)
    assert len(b) == 3
    assert [b.ids(i) for i in range(3)] == [[5, 4], [3, 2], [1]]
    assert b.push(5) is None
    assert b.push(4) == 0


def test_capacity_zero_is_an_error():
    with pytest.raises(ValueError, match="capacity must be >= 1"):
        GradBuckets([1, 2], 0)
