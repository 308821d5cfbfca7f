"""Model check of the NEXT-3 peer-memory allreduce protocol (peer_reduce.cu)
on CPU threads.  P ranks repeat, with random delays and slow readers:
  publish:  write the own partial (one value per chunk) into the single PUB
            region, then signal PUB epoch e to every peer's pad;
  reduce-scatter: wait until every PUB word of the own pad reaches e, sum
            the own chunk over all ranks' PUB regions (rank order), write it
            into the single RED region, signal RED epoch e to every peer;
  all-gather: wait until every RED word reaches e, read every chunk from its
            owner's RED region.
One region of each kind and no extra barrier must never let a rank overwrite
a region a peer is still reading: every rank must get the exact sum every
round.  Negative controls drop one of the two waits and must expose a race.
(The CUDA kernels run bit-exactly at one rank on the GPU; this checks the
multi-rank ordering argument itself.)"""
import random
import threading
import time

import pytest


def _run(P, rounds, seed, skip_rs_wait=False, skip_ag_wait=False):
    rng = random.Random(seed)
    delays = [[rng.random() * 1e-4 for _ in range(8 * rounds * (P + 2))] for _ in range(P)]
    pub = [[0.0] * P for _ in range(P)]            # pub[rank][chunk]
    red = [0.0] * P                                  # red[rank] = the rank's chunk of the sum
    pad_pub = [[0] * P for _ in range(P)]            # pad_pub[owner][writer]
    pad_red = [[0] * P for _ in range(P)]
    cv = threading.Condition()
    errors = []
    done = [0] * P

    # the negative controls skew the ranks by milliseconds (rank r starts each
    # round r x 2 ms late), so a missing wait shows up whatever the host load
    skew = 2e-3 if (skip_rs_wait or skip_ag_wait) else 0.0

    def rank(r):
        d = iter(delays[r])
        for it in range(rounds):
            e = it + 1
            time.sleep(next(d) + skew * r)
            for c in range(P):                       # publish (fused into the chunk sum)
                pub[r][c] = float((1 + r + 10 * it) * (c + 1))
                time.sleep(next(d) / 4)
            with cv:                                 # last block: signal PUB = e to every peer
                for q in range(P):
                    pad_pub[q][r] = e
                cv.notify_all()
                if not skip_rs_wait:
                    cv.wait_for(lambda: all(pad_pub[r][q] >= e for q in range(P)))
            s = 0.0
            for q in range(P):                       # reduce-scatter: own chunk, rank order
                s += pub[q][r]
                time.sleep(next(d) * (1 + r) / 4)    # slower ranks read slower
            red[r] = s
            with cv:
                for q in range(P):
                    pad_red[q][r] = e
                cv.notify_all()
                if not skip_ag_wait:
                    cv.wait_for(lambda: all(pad_red[r][q] >= e for q in range(P)))
            out = []
            for c in range(P):                       # all-gather from every owner's RED region
                out.append(red[c])
                time.sleep(next(d) * (1 + r) / 4)
            want = [float(sum((1 + q + 10 * it) * (c + 1) for q in range(P))) for c in range(P)]
            if out != want:
                errors.append((r, it))
        done[r] = rounds

    th = [threading.Thread(target=rank, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert done == [rounds] * P, "a rank thread did not finish"
    return errors


@pytest.mark.parametrize("P", [2, 3, 8])
def test_reduce_scatter_all_gather_single_regions(P):
    assert _run(P, 30, seed=P) == []


@pytest.mark.parametrize("which", ["rs", "ag"])
def test_model_detects_a_missing_wait(which):
    """Sanity of the model: without the reduce-scatter wait a rank sums
    partials not yet published; without the all-gather wait it reads chunks
    not yet reduced -- both must show up as wrong sums."""
    bad = []
    for seed in range(6):
        bad += _run(4, 12, seed=100 + seed, skip_rs_wait=(which == "rs"), skip_ag_wait=(which == "ag"))
        if bad:
            break
    assert bad, f"the model failed to expose the race without the {which} wait"
