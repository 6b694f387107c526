"""Host-side lane bookkeeping of the device caches: the parent lists behind gather_lanes /
keep_lanes / permute_lanes, with the reference's checks and error types
(DecoderState, model.hpp:291-325).  CPU only."""
import numpy as np
import pytest

import paper_2105_04779_b200 as E


def test_gather_indices_repeat_and_resize():
    assert E.gather_lane_indices([2, 2, 0], 3).tolist() == [2, 2, 0]
    assert E.gather_lane_indices([1], 4).tolist() == [1]


@pytest.mark.parametrize("bad,err", [([], E.StateError), ([3], E.ParamError), ([-1, 0], E.ParamError)])
def test_gather_indices_errors(bad, err):
    with pytest.raises(err):
        E.gather_lane_indices(bad, 3)


def test_keep_indices():
    assert E.keep_lane_indices([True, False, True, True], 4).tolist() == [0, 2, 3]
    with pytest.raises(E.ParamError):
        E.keep_lane_indices([True, False], 3)
    with pytest.raises(E.StateError):
        E.keep_lane_indices([False, False], 2)


def test_permute_indices():
    assert E.permute_lane_indices([2, 0, 1], 3).tolist() == [2, 0, 1]
    for bad in ([0, 0, 1], [0, 1], [0, 1, 3]):
        with pytest.raises(E.ParamError):
            E.permute_lane_indices(bad, 3)
