"""Oracle: device-memory allocator models and their replay over a schedule.

Virtual addressing (§4):
  "we map small physical memory chunks with constant size to a consecutive
  virtual address.  Once a variable is cleared ... we release a virtual
  address and cache physical memories for the future requests".
  m_a = k·m_c with k = ⌈m_r / m_c⌉, IF = m_a − m_r < m_c   (Eq.1)
  IF_max < N_max·m_c                                       (Eq.2)
  Chunks are taken from a FIFO of free chunks (oldest released first); the
  pool holds ⌊B_p / m_c⌋ chunks; a request fails iff fewer than k are free.

Caching best-fit arena (the frameworks' default):
  requests are rounded up to `align`; the smallest cached free block >= s is
  reused (ties: lowest address) and split, the remainder staying cached in
  the same segment; otherwise a new segment of exactly s is carved from the
  untouched tail of the capacity; otherwise DeviceOOM — even when the free
  bytes in total would suffice (external fragmentation).  A freed
  block coalesces only with address-adjacent free blocks of its own segment.
First-fit: as best-fit but the lowest-address free block >= s is taken.

Replay order per f_i (reading Z9):
  free(wait_out[i]) -> alloc(in[i]) -> [f_i] -> free(free[i]); end: free(end_wait).
"""


class DeviceOOM(Exception):
    def __init__(self, fn, var, request, free_bytes):
        super().__init__(f"DeviceOOM at f{fn}: var {var} needs {request}, free {free_bytes}")
        self.fn, self.var, self.request, self.free_bytes = fn, var, request, free_bytes


class AllocError(Exception):
    pass


class VAPool:
    """Chunk pool + per-allocation virtual spans."""

    def __init__(self, chunk_bytes, phys_bytes):
        self.m_c = chunk_bytes
        self.n_chunks = phys_bytes // chunk_bytes
        self.free_q = list(range(self.n_chunks))   # FIFO, oldest released first
        self.live = {}                              # handle -> (m_r, chunks)
        self.next_handle = 0
        self.freed = set()
        self.peak_chunks = 0
        self.if_peak = 0
        self.n_max = 0

    def alloc(self, m_r):
        k = -(-m_r // self.m_c)                      # k = ⌈m_r / m_c⌉
        if len(self.free_q) < k:
            return None
        chunks = self.free_q[:k]
        self.free_q = self.free_q[k:]
        h = self.next_handle
        self.next_handle += 1
        self.live[h] = (m_r, chunks)
        mapped = self.n_chunks - len(self.free_q)
        self.peak_chunks = max(self.peak_chunks, mapped)
        self.if_peak = max(self.if_peak, self.internal_frag())
        self.n_max = max(self.n_max, len(self.live))
        return h

    def free(self, h):
        if h in self.freed:
            raise AllocError("DoubleFree")
        if h not in self.live:
            raise AllocError("UnknownHandle")
        _, chunks = self.live.pop(h)
        self.freed.add(h)
        self.free_q.extend(chunks)

    def internal_frag(self):
        """Σ over live allocations of m_a − m_r (Eq.1 summed)."""
        return sum(len(c) * self.m_c - m_r for (m_r, c) in self.live.values())

    def free_bytes(self):
        return len(self.free_q) * self.m_c

    def chunks_of(self, h):
        return list(self.live[h][1])


class Arena:
    """Caching best-fit (or first-fit) allocator over one capacity range."""

    def __init__(self, capacity, align=512, policy="best"):
        self.capacity = capacity
        self.align = align
        self.policy = policy
        self.tail = 0                 # untouched capacity starts here
        self.blocks = []              # [start, size, segment, free(bool), handle]
        self.live = {}
        self.freed = set()
        self.next_handle = 0
        self.allocated = 0
        self.peak_allocated = 0

    def _round(self, n):
        return -(-n // self.align) * self.align

    def alloc(self, m_r):
        s = self._round(m_r)
        cands = [blk for blk in self.blocks if blk[3] and blk[1] >= s]
        if cands:
            if self.policy == "best":
                blk = min(cands, key=lambda x: (x[1], x[0]))
            else:
                blk = min(cands, key=lambda x: x[0])
            if blk[1] > s:
                rest = [blk[0] + s, blk[1] - s, blk[2], True, None]
                self.blocks.insert(self.blocks.index(blk) + 1, rest)
            blk[1] = s
            blk[3] = False
        elif self.capacity - self.tail >= s:
            seg = self.tail
            blk = [self.tail, s, seg, False, None]
            self.blocks.append(blk)
            self.tail += s
        else:
            return None
        h = self.next_handle
        self.next_handle += 1
        blk[4] = h
        self.live[h] = blk
        self.allocated += s
        self.peak_allocated = max(self.peak_allocated, self.allocated)
        return h

    def free(self, h):
        if h in self.freed:
            raise AllocError("DoubleFree")
        if h not in self.live:
            raise AllocError("UnknownHandle")
        blk = self.live.pop(h)
        self.freed.add(h)
        self.allocated -= blk[1]
        blk[3] = True
        blk[4] = None
        # coalesce with address-adjacent free blocks of the same segment
        self.blocks.sort(key=lambda x: x[0])
        merged = []
        for x in self.blocks:
            if merged and merged[-1][3] and x[3] and merged[-1][2] == x[2] \
                    and merged[-1][0] + merged[-1][1] == x[0]:
                merged[-1][1] += x[1]
            else:
                merged.append(x)
        self.blocks = merged

    def free_bytes(self):
        """Cached free bytes plus untouched capacity."""
        return sum(x[1] for x in self.blocks if x[3]) + (self.capacity - self.tail)

    def largest_free(self):
        return max([x[1] for x in self.blocks if x[3]] + [self.capacity - self.tail])

    def offset_of(self, h):
        return self.live[h][0]


def replay(g, sch, mode, chunk_bytes=40 << 20, phys_bytes=None, align=512):
    """Replay a schedule's alloc/free calls through one allocator model.

    Returns stats {peak_phys, peak_alloc, if_peak, n_max, oom} and the
    placement of every arrival (chunk list or arena offset), in call order.
    `phys_bytes` is the swap pool B_p (pinned variables live outside it)."""
    if mode == "va":
        A = VAPool(chunk_bytes, phys_bytes)
    elif mode in ("best", "first"):
        A = Arena(phys_bytes, align, mode)
    else:
        raise ValueError(mode)
    handle = {}
    placements = []
    oom = None
    n = len(sch.ins)
    try:
        for i in range(n):
            for v in sch.wait_out[i]:
                A.free(handle.pop(v))
            for v, _kind in sch.ins[i]:
                h = A.alloc(g.var_bytes[v])
                if h is None:
                    raise DeviceOOM(i, v, g.var_bytes[v], A.free_bytes())
                handle[v] = h
                placements.append((i, v, A.chunks_of(h) if mode == "va" else A.offset_of(h)))
            for v in sch.free[i]:
                A.free(handle.pop(v))
        for v in sch.end_wait:
            A.free(handle.pop(v))
    except DeviceOOM as e:
        oom = {"fn": e.fn, "var": e.var, "request": e.request, "free_bytes": e.free_bytes}
    if mode == "va":
        stats = {"peak_phys": A.peak_chunks * A.m_c, "if_peak": A.if_peak, "n_max": A.n_max}
    else:
        stats = {"peak_phys": A.tail, "peak_alloc": A.peak_allocated}
    stats["oom"] = oom
    return stats, placements
