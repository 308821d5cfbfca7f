"""Model check of the NEXT-3 peer-memory allreduce protocol (peer_reduce.cu)
on CPU threads: P ranks repeat {publish own partial into slot (epoch+1)&1 of
the local exchange buffer; barrier: epoch += 1, signal every peer's pad slot
`rank`, wait for all pads; sum slot epoch&1 of every rank's buffer in rank
order} with random delays.  Two alternating slots and ONE barrier per
allreduce must never let a rank overwrite a slot a peer is still reading:
every rank must get the exact sum every round.  (The CUDA kernels are
exercised bit-exactly at one rank on the GPU; this checks the multi-rank
ordering argument itself.)"""
import random
import threading

import pytest


def _run(P, rounds, seed):
    rng = random.Random(seed)
    delays = [[rng.random() * 1e-4 for _ in range((3 + P) * rounds)] for _ in range(P)]
    bufs = [[[0.0], [0.0]] for _ in range(P)]          # [rank][slot] -> value
    pads = [[0] * P for _ in range(P)]                  # pads[owner][writer]
    epoch = [0] * P
    cv = threading.Condition()
    errors = []
    done = [0] * P

    def rank(r):
        import time
        d = iter(delays[r])
        for it in range(rounds):
            val = float(1 + r + 10 * it)
            time.sleep(next(d))
            bufs[r][(epoch[r] + 1) & 1][0] = val            # publish (fused into the chunk reduce)
            time.sleep(next(d))
            with cv:                                         # barrier
                epoch[r] += 1
                e = epoch[r]
                for q in range(P):
                    pads[q][r] = e
                cv.notify_all()
                cv.wait_for(lambda: all(pads[r][q] >= e for q in range(P)))
            time.sleep(next(d))
            tot = 0.0
            order = range(P) if r % 2 == 0 else reversed(range(P))   # the kernel reads 0..P-1; the
            for q in order:                                           # protocol must not depend on it
                tot += bufs[q][e & 1][0]
                time.sleep(next(d) * (1 + r) / 4)            # slower ranks read slower: peers race ahead
            want = float(sum(1 + q + 10 * it for q in range(P)))
            if tot != want:
                errors.append((r, it, tot, want))
        done[r] = rounds

    th = [threading.Thread(target=rank, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=60)
    assert done == [rounds] * P, "a rank thread did not finish"
    return errors


@pytest.mark.parametrize("P", [2, 3, 8])
def test_two_slots_one_barrier_suffice(P):
    assert _run(P, 40, seed=P) == []


def test_model_detects_a_single_slot():
    """Sanity of the model itself: with ONE slot (no alternation) a fast rank
    overwrites its partial while a slow peer still reads it, and the model
    sees wrong sums."""
    bad = _run_single_slot(4, 40, seed=1)
    assert bad, "the model failed to expose the single-slot race"


def _run_single_slot(P, rounds, seed):
    import time
    rng = random.Random(seed)
    buf = [0.0] * P
    pads = [[0] * P for _ in range(P)]
    epoch = [0] * P
    cv = threading.Condition()
    errors = []

    def rank(r):
        for it in range(rounds):
            time.sleep(rng.random() * 1e-4)
            buf[r] = float(1 + r + 10 * it)
            with cv:
                epoch[r] += 1
                e = epoch[r]
                for q in range(P):
                    pads[q][r] = e
                cv.notify_all()
                cv.wait_for(lambda: all(pads[r][q] >= e for q in range(P)))
            tot = 0.0
            for q in reversed(range(P)):                     # read the fast rank 0 last
                tot += buf[q]
                time.sleep((r + 1) * 2e-4)                   # slow readers: peers race ahead
            if tot != float(sum(1 + q + 10 * it for q in range(P))):
                errors.append((r, it))

    th = [threading.Thread(target=rank, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=60)
    return errors
