"""Engine bucketing: the greedy reverse-order packing of
engine.cpp:76-95, pinned on the reference's own engine tests."""
import pytest

from paper_2107_01499_b200._lib import Error
from paper_2107_01499_b200.engine import plan_buckets


def test_greedy_reverse_order_packing_respects_capacity():
    # test_engine.cpp:65-83: mlp(d=4, hidden=8) layer sizes 32, 8, 8, 1 floats, capacity 40 B
    b = plan_buckets([32, 8, 8, 1], 40)
    assert [x.layers for x in b] == [[3, 2], [1], [0]]
    assert b[0].trigger_layer == 2  # last member to finish backward
    assert b[0].elements == 9 and b[2].elements == 32
    assert [x.id for x in b] == [0, 1, 2]


def test_fusion_disabled_one_bucket_per_layer():
    # test_engine.cpp:85-93
    b = plan_buckets([32, 8, 8, 1], 40, fusion=False)
    assert [x.layers for x in b] == [[3], [2], [1], [0]]


def test_oversized_layer_gets_its_own_bucket_and_default_capacity():
    # a layer above the capacity still opens (and fills) one bucket; 8 MiB default (engine.hpp:58)
    b = plan_buckets([3 << 20, 1 << 20, 1 << 20], 8 << 20)
    assert [x.layers for x in b] == [[2, 1], [0]]
    b = plan_buckets([10], 4)
    assert [x.layers for x in b] == [[0]] and b[0].elements == 10


def test_no_layers_is_an_error():
    with pytest.raises(Error):
        plan_buckets([], 40)
