"""Online monitor: the oracle pinned by hand-worked cases,
then the C-ABI implementation bit-exact against it on random traces."""
import random
from fractions import Fraction

import pytest

from oracle import monitor as OM

MS = 1_000_000
W = 300 * MS                     # P:597 default window
BETA = Fraction(3, 2)            # P:597 default β


def test_oracle_no_queueing_stays_latency():
    # every request runs immediately: L_req == L_exec, ratio 1 < β
    reqs = [(t * MS, 40 * MS, 40 * MS) for t in range(0, 900, 10)]
    trace, n = OM.policy_trace(reqs, W, BETA)
    assert trace == [OM.LATENCY] * 3 and n == 0


def test_oracle_queueing_spike_switches_and_back():
    # window 0 light (ratio 1.2), window 1 heavy (ratio 4: queueing 3x exec), window 2 light again
    reqs = [(100 * MS, 12, 10), (350 * MS, 40, 10), (500 * MS, 40, 10), (700 * MS, 10, 10)]
    trace, n = OM.policy_trace(reqs, W, BETA)
    assert trace == [OM.LATENCY, OM.THROUGHPUT, OM.LATENCY] and n == 2


def test_oracle_ratio_equal_beta_is_latency_and_means_not_sums():
    # means: req (10+20)/2 = 15, exec (10+10)/2 = 10 → ratio exactly 1.5 = β → latency
    trace, _ = OM.policy_trace([(1, 10, 10), (2, 20, 10)], W, BETA, initial=OM.THROUGHPUT)
    assert trace == [OM.LATENCY]
    # ratio of means, not mean of ratios: (1 + 99)/2 / ((1 + 99)/2) = 1 though one request alone has ratio 99
    trace, _ = OM.policy_trace([(1, 99, 1), (2, 1, 99)], W, BETA)
    assert trace == [OM.LATENCY]


def test_oracle_empty_window_keeps_policy():
    reqs = [(10, 30, 10), (2 * W + 5, 30, 10)]
    trace, n = OM.policy_trace(reqs, W, BETA)
    assert trace == [OM.THROUGHPUT, OM.THROUGHPUT, OM.THROUGHPUT] and n == 1


@pytest.fixture(scope="module")
def api():
    from paper_2604_10180_b200 import api as A
    return A


def test_monitor_defaults_and_errors(api):
    from paper_2604_10180_b200 import _kd as K
    m = api.Monitor()
    assert m.poll(0) == (K.KD_OBJ_LATENCY, 0)
    m.record(W + 1, 10, 10)
    assert m.poll(2 * W)[0] == K.KD_OBJ_LATENCY
    with pytest.raises(K.KdError):
        m.record(W - 1, 10, 10)  # that window was already evaluated


@pytest.mark.parametrize("seed", range(20))
def test_monitor_matches_oracle_random_traces(api, seed):
    rnd = random.Random(seed)
    window = rnd.choice([30 * MS, 300 * MS, 1500 * MS])
    beta = Fraction(rnd.choice([11, 15, 30]), 10)
    n = rnd.randint(1, 300)
    t = 0
    reqs = []
    for _ in range(n):
        t += rnd.randint(0, 40 * MS)
        exe = rnd.randint(1, 50 * MS)
        reqs.append((t, exe + rnd.choice([0, 0, rnd.randint(0, 200 * MS)]), exe))
    horizon = (t // window + 1) * window
    ref, ref_sw = OM.policy_trace(reqs, window, beta, horizon_ns=horizon)
    m = api.Monitor(window, (beta.numerator, beta.denominator))
    got = []
    i = 0
    for w in range(horizon // window):
        while i < n and reqs[i][0] < (w + 1) * window:   # arrivals of window w, in time order
            m.record(*reqs[i])
            i += 1
        p, sw = m.poll((w + 1) * window)
        got.append(p)
    assert got == ref and sw == ref_sw
