"""The runtime's ONE residency policy (memplan::ChunkBufferPool through the
ptk_pool_* C-ABI; include/memplan/policy.hpp) -- the decisions the simulator,
the device executor and the training-time chunk pool all make -- and the
planner CLI in process (ptk_memplan_run). No GPU needed: these are host code
in libptk.so.

Rules under test (proj/src/sim.cpp:275-343,427-451): lowest free slot first;
else evict the idle resident non-persistent chunk whose next use is farthest
(forward position c, backward 2N-c+1), strictly later than the incoming
chunk's, never a pinned chunk, lower id on ties; arriving chunks are not
evictable; a release frees the slot."""
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2406_08334_b200 import _native as nat  # noqa: E402
from paper_2406_08334_b200 import planner  # noqa: E402


def test_free_slots_then_farthest_next_use_eviction():
    # 6 chunks (0-based 0..5), chunk 0 persistent, 2 buffers; N = 6
    p = nat.BufferPool(6, 1, 2)
    assert p.residency(0) == 2 and p.slot_of(0) == -1  # persistent: resident, no slot
    assert p.grant(1, 2) == (0, None)
    assert p.grant(2, 3) == (1, None)
    # both slots hold ARRIVING chunks: nothing can be evicted yet
    assert p.grant(3, 4) is None
    p.arrived(1)
    p.arrived(2)
    # forward position 4 (0-based chunk 3): next uses are the backward positions
    # 2N-c: chunk 1 -> 11, chunk 2 -> 10; farthest = chunk 1
    assert p.grant(3, 4, pinned=(3, 2)) == (0, 1)
    assert p.residency(1) == 0 and p.chunk_in_slot(0) == 3
    p.arrived(3)
    # pinned chunks are never evicted
    assert p.grant(4, 5, pinned=(4, 3, 2)) is None


def test_strictly_later_rule_refuses_a_prefetch():
    p = nat.BufferPool(4, 0, 1)
    assert p.grant(2, 3) == (0, None)
    p.arrived(2)
    # backward phase, position 5 (= backward of 0-based chunk 2 at 2N-c = 6):
    # chunk 2's next use (6) is SOONER than chunk 1's (7): no eviction for chunk 1
    assert p.grant(1, 5) is None
    # at position 7 chunk 2 has no use left: it gives way
    assert p.grant(1, 7) == (0, 2)


def test_ties_go_to_the_lower_chunk_and_release_frees_the_slot():
    p = nat.BufferPool(5, 0, 2)
    for c, now in ((3, 4), (4, 5)):
        p.grant(c, now)
        p.arrived(c)
    # position 8: chunks 3 and 4 are past their backward uses (7 and 6), both
    # "never" -> the lower id gives way to chunk 1 (backward use at 9)
    assert p.grant(1, 8) == (0, 3)
    p.arrived(1)
    # an incoming chunk with no use left never evicts anything on a prefetch ...
    assert p.grant(2, 11) is None
    # ... but a demand fetch (needed now) takes the farthest candidate
    assert p.grant(2, 11, pinned=(2,), demand=True) == (0, 1)
    p.arrived(2)
    assert p.release(4) == 1
    assert p.residency(4) == 0 and p.chunk_in_slot(1) is None
    assert p.grant(1, 11) == (1, None)


def test_pool_errors_are_loud():
    p = nat.BufferPool(3, 1, 1)
    with pytest.raises(nat.PtkError):
        p.grant(0, 1)  # persistent chunk
    with pytest.raises(nat.PtkError):
        p.arrived(2)  # was not arriving
    with pytest.raises(nat.PtkError):
        nat.BufferPool(2, 3, 1)  # n_persist > n_chunk


def test_memplan_in_process_matches_the_cli(tmp_path):
    """ptk_memplan_run (memplan::run_cli in libptk.so) writes exactly what the
    memplan binary writes, and reports usage errors with exit code 2."""
    trace = str(tmp_path / "t.json")
    planner.trace_file(planner.TRACE_ARGS["gpt2-1b_b2"], trace)
    args = ["plan", "--trace", trace, "--hw", "a100x1"]
    rc, out, err = nat.memplan_run(args)
    binary = os.path.join(REPO, "build", "memplan")
    if os.path.exists(binary):
        r = subprocess.run([binary] + args, capture_output=True, text=True)
        assert (rc, out) == (r.returncode, r.stdout)
    assert rc == 0 and '"n_persist"' in out
    rc, out, err = nat.memplan_run(["plan"])
    assert rc == 2 and err
