"""Pins for the reference block manager (oracle/block_manager.py) from the paper's worked
examples (P:N = PAPER.md line N), plus a conservation-law fuzz."""
import random

import pytest

from oracle.block_manager import BlockManager, OutOfBlocks


def fig6_manager():
    # Force the free list to hand out 7, 1, 3 first, as in Fig.6.
    order = [7, 1, 3] + [b for b in range(8) if b not in (7, 1, 3)]
    return BlockManager(8, 4, initial_order=order)


def test_fig6_block_table_translation():
    """7-token prompt, B = 4 -> logical {0,1} -> physical {7,1}; first decode
    fills the last slot of block 1; the second needs new block 3."""
    m = fig6_manager()
    h = m.allocate(7)
    assert m.block_table(h) == [7, 1]
    assert [f for _, f in m.tables[h]] == [4, 3]
    prompt_slots = [m.block_table(h)[t // 4] * 4 + t % 4 for t in range(7)]
    assert prompt_slots == [28, 29, 30, 31, 4, 5, 6]
    assert m.append_slot(h) == ("inplace", 7, None)
    assert m.append_slot(h) == ("newblock", 12, None)
    assert m.block_table(h) == [7, 1, 3]
    m.check_conservation()


def test_parallel_sampling_copy_on_write():
    """Fig.8: samples share 7,1 with refcount 2; A1's append copies block 1
    into new block 3 and drops refcount(1) to 1; A2 then writes block 1 in place."""
    m = fig6_manager()
    a1 = m.allocate(7)
    a2 = m.fork(a1)
    assert m.ref[7] == 2 and m.ref[1] == 2
    kind, slot, cow = m.append_slot(a1)
    assert kind == "cow" and cow == (1, 3) and slot == 3 * 4 + 3
    assert m.ref[1] == 1 and m.ref[3] == 1 and m.ref[7] == 2
    assert m.append_slot(a2) == ("inplace", 1 * 4 + 3, None)
    assert m.block_table(a1) == [7, 3] and m.block_table(a2) == [7, 1]
    m.check_conservation()


def test_beam_search_fig9():
    """Fig.9: before the step the candidates hold [0,1,3,2], [0,1,3,6],
    [0,1,3,7], [0,4,5,8]; the new top-4 all descend from candidates 1 and 2; freeing
    candidates 0 and 3 frees exactly {2,4,5,8}; new blocks 9-12 are allocated; all
    share 0,1,3, new candidates 0,1 share 6 and 2,3 share 7.  Only these text-pinned
    facts are asserted."""
    B = 2
    order = [0, 1, 4, 3, 5, 2, 6, 7, 8] + list(range(9, 16))
    m = BlockManager(16, B, initial_order=order)

    def grow(h, n):
        for _ in range(n):
            m.append_slot(h)

    c0 = m.allocate(B)
    c3 = m.fork(c0)
    grow(c0, B); grow(c3, B); grow(c0, B); grow(c3, B)
    c1, c2 = m.fork(c0), m.fork(c0)
    grow(c0, B); grow(c1, B); grow(c2, B); grow(c3, B)
    assert [m.block_table(c) for c in (c0, c1, c2, c3)] == [[0, 1, 3, 2], [0, 1, 3, 6], [0, 1, 3, 7], [0, 4, 5, 8]]
    n0, n1, n2, n3 = m.fork(c1), m.fork(c1), m.fork(c2), m.fork(c2)
    freed = set()
    before = set(m.free_list)
    for c in (c0, c1, c2, c3):
        m.free(c)
    freed = set(m.free_list) - before
    assert freed == {2, 4, 5, 8}
    cows = [m.append_slot(n)[2] for n in (n0, n1, n2, n3)]
    assert cows == [None] * 4  # every old block is full: no copy
    tables = [m.block_table(n) for n in (n0, n1, n2, n3)]
    assert sorted(t[-1] for t in tables) == [9, 10, 11, 12]
    assert all(t[:3] == [0, 1, 3] for t in tables)
    assert tables[0][3] == tables[1][3] == 6 and tables[2][3] == tables[3][3] == 7
    m.check_conservation()


def test_waste_within_one_block_and_out_of_blocks():
    """waste per request <= one block; OutOfBlocks on an empty free list."""
    m = BlockManager(4, 4)
    h = m.allocate(5)
    assert len(m.block_table(h)) * 4 - m.num_tokens(h) <= 3
    m.allocate(8)
    with pytest.raises(OutOfBlocks):
        m.allocate(1)
    with pytest.raises(OutOfBlocks):
        for _ in range(4):
            m.append_slot(h)


def test_fork_free_identity_and_double_free():
    m = BlockManager(10, 4)
    h = m.allocate(9)
    ref0 = list(m.ref)
    c = m.fork(h)
    assert m.free(c) == 0
    assert m.ref == ref0
    with pytest.raises(KeyError):
        m.free(c)


def test_fuzz_conservation():
    """Random allocate/append/fork/free: conservation laws after every op."""
    rs = random.Random(18)
    m = BlockManager(64, 4, initial_order=rs.sample(range(64), 64))
    live = []
    for _ in range(20000):
        op = rs.random()
        try:
            if op < 0.15 or not live:
                live.append(m.allocate(rs.randint(1, 12)))
            elif op < 0.7:
                h = rs.choice(live)
                kind, slot, cow = m.append_slot(h)
                if cow is not None:
                    assert m.ref[cow[1]] == 1 and m.ref[cow[0]] >= 1
            elif op < 0.85:
                live.append(m.fork(rs.choice(live)))
            else:
                h = live.pop(rs.randrange(len(live)))
                m.free(h)
        except OutOfBlocks:
            h = live.pop(rs.randrange(len(live)))
            m.free(h)
        m.check_conservation()
