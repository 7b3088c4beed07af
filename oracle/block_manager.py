"""Plain-Python reference of the paper's KV block manager.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  It is the oracle for the product's
host allocator (``pa_alloc_*`` in libpagedattn.so): tests drive both with the same
operation sequence and compare every table, refcount and copy-on-write directive.

Follows (P:N = PAPER.md line N):
- logical blocks filled left to right, a new physical block only when the last is full
  (Fig.6 ``block-table-translation``);
- reference counts and block-granular copy-on-write (Fig.8
  ``parallel-decoding``);
- ``fork`` / ``append`` / ``free``; freeing returns blocks whose count
  reaches zero (Fig.9 ``beam-search``).
The SPEC's operation contracts fix most details the paper leaves open:
double free is an error, OutOfBlocks when the free list is empty (S:132,
S:155).  The free list is a FIFO queue, NOT the SPEC's LIFO stack: Fig.9's
text frees blocks 2, 4, 5, 8 and then allocates blocks 9-12, which only a
queue that hands out never-used blocks before recycled ones reproduces (DESIGN.md
reading c19).
"""
from __future__ import annotations

from collections import deque


class OutOfBlocks(Exception):
    pass


class BlockManager:
    def __init__(self, num_blocks: int, block_size: int, initial_order=None):
        """``initial_order``: physical ids in the order they will be handed out (the first
        element is allocated first).  Default: 0, 1, ..., num_blocks-1."""
        if num_blocks <= 0 or block_size <= 0:
            raise ValueError("num_blocks and block_size must be positive")
        self.B = block_size
        self.num_blocks = num_blocks
        order = list(range(num_blocks)) if initial_order is None else list(initial_order)
        if sorted(order) != list(range(num_blocks)):
            raise ValueError("initial_order must be a permutation of range(num_blocks)")
        # FIFO queue: allocate from the front, freed blocks join the back
        self.free_list = deque(order)
        self.ref = [0] * num_blocks
        self.tables = {}  # handle -> list of [block, filled]
        self._next = 0

    # -- helpers -------------------------------------------------------------------
    def _pop(self) -> int:
        if not self.free_list:
            raise OutOfBlocks()
        b = self.free_list.popleft()
        assert self.ref[b] == 0
        self.ref[b] = 1
        return b

    def num_free(self) -> int:
        return len(self.free_list)

    def num_tokens(self, h: int) -> int:
        return sum(f for _, f in self.tables[h])

    # -- S:128 allocate --------------------------------------------------------------
    def allocate(self, num_tokens: int) -> int:
        if num_tokens <= 0:
            raise ValueError("num_tokens must be positive")
        n = -(-num_tokens // self.B)
        if n > len(self.free_list):
            raise OutOfBlocks()
        entries = []
        left = num_tokens
        for _ in range(n):
            f = min(self.B, left)
            entries.append([self._pop(), f])
            left -= f
        h = self._next
        self._next += 1
        self.tables[h] = entries
        return h

    def can_allocate(self, num_tokens: int, watermark: int = 0) -> bool:
        return len(self.free_list) >= -(-num_tokens // self.B) + watermark

    # -- S:148 append_slot -----------------------------------------------------------
    def append_slot(self, h: int):
        """Returns (kind, slot, cow) with kind in {"inplace", "newblock", "cow"},
        slot = physical_block * B + offset of the appended token, cow = (src, dst) or None."""
        t = self.tables[h]
        last = t[-1] if t else None
        if last is None or last[1] == self.B:
            b = self._pop()
            t.append([b, 1])
            return "newblock", b * self.B, None
        blk, filled = last
        if self.ref[blk] == 1:
            last[1] += 1
            return "inplace", blk * self.B + filled, None
        # shared partial last block: copy-on-write
        dst = self._pop()
        self.ref[blk] -= 1
        last[0] = dst
        last[1] += 1
        return "cow", dst * self.B + filled, (blk, dst)

    # -- S:161 fork -----------------------------------------------------------------
    def fork(self, parent: int) -> int:
        entries = [[b, f] for b, f in self.tables[parent]]
        for b, _ in entries:
            self.ref[b] += 1
        h = self._next
        self._next += 1
        self.tables[h] = entries
        return h

    # -- S:171 free -----------------------------------------------------------------
    def free(self, h: int) -> int:
        if h not in self.tables:
            raise KeyError("double free or unknown sequence")
        freed = 0
        for b, _ in self.tables.pop(h):
            if self.ref[b] <= 0:
                raise RuntimeError("refcount underflow")
            self.ref[b] -= 1
            if self.ref[b] == 0:
                self.free_list.append(b)
                freed += 1
        return freed

    # -- export ---------------------------------------------------------------------
    def block_table(self, h: int):
        return [b for b, _ in self.tables[h]]

    def export(self, handles, W: int):
        rows, lens = [], []
        for h in handles:
            ids = self.block_table(h)
            if len(ids) > W:
                raise ValueError("W too small")
            rows.append(ids + [-1] * (W - len(ids)))
            lens.append(self.num_tokens(h))
        return rows, lens

    def check_conservation(self) -> None:
        """Refcount conservation law and pool conservation."""
        count = [0] * self.num_blocks
        for entries in self.tables.values():
            for b, _ in entries:
                count[b] += 1
        assert count == self.ref, "refcount conservation violated"
        assert len(self.free_list) + sum(1 for r in self.ref if r > 0) == self.num_blocks
        assert set(self.free_list) == {b for b in range(self.num_blocks) if self.ref[b] == 0}
        for entries in self.tables.values():
            for b, f in entries[:-1]:
                assert f == self.B
            if entries:
                assert 1 <= entries[-1][1] <= self.B
