"""Impact-zone host logic on CPU: distribute_zones (response.cpp:164-182)
behind the C-ABI (weft_distribute_zones), the known answers of
proj/tests/test_response.cpp:144-172 and random cases against a direct
restatement of the greedy loop."""
import numpy as np


def greedy(sizes, devices):
    """response.cpp:164-182, restated: stable descending sort by vertex
    count, each zone to the least-loaded device (lowest index on ties)."""
    order = sorted(range(len(sizes)), key=lambda z: -sizes[z])
    out = [[] for _ in range(devices)]
    load = [0] * devices
    for z in order:
        best = min(range(devices), key=lambda d: (load[d], d))
        out[best].append(z)
        load[best] += sizes[z]
    return out


def test_distribute_zones_known_answers():
    from paper_2008_00409_b200 import weft
    assert [len(a) for a in weft.distribute_zones([3, 3, 3, 3], 4)] == [1, 1, 1, 1]
    assert weft.distribute_zones([8, 1, 1, 1, 1], 2) == [[0], [1, 2, 3, 4]]
    a = weft.distribute_zones([100], 4)
    assert a[0] == [0] and all(x == [] for x in a[1:])
    assert weft.distribute_zones([], 3) == [[], [], []]


def test_distribute_zones_random():
    from paper_2008_00409_b200 import weft
    rng = np.random.default_rng(7)
    for _ in range(50):
        n = int(rng.integers(1, 60))
        sizes = rng.integers(1, 40, n).tolist()
        d = int(rng.integers(1, 9))
        assert weft.distribute_zones(sizes, d) == greedy(sizes, d)
