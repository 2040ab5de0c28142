"""Pure-Python restatements of numpy's float64 association orders -- TEST
INFRASTRUCTURE (the checker for the order contract the CUDA kernels follow,
see paper_1509_05194_b200/csrc/common.cuh).  Pinned against numpy itself in
tests/test_np_order.py and against the reference outputs in tests/golden.

* pairwise(a): numpy's pairwise_sum (numpy/_core/src/umath/loops_utils.h.src):
  n < 8 sequential from 0.0; n <= 128 eight interleaved accumulators folded
  ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the tail; above 128 split at
  n/2 rounded down to a multiple of 8 and recurse.  Used by every contiguous
  row sum in the reference (e.g. clustering.py:142-144, codebook.py:300) and by
  1-D .mean() (clustering.py:187).
* reduceat_segment(rows): np.add.reduceat along axis 0 = first row +
  pairwise(rest) per column (clustering.py:160).
* einsum_sq(c): einsum('mkd,mkd->mk') = SSE2 two-lane mul+add with blocks of
  four vectors consumed high-to-low (codebook.py:129, 237, 260).
* axis-0 .mean(): sequential from the first row (clustering.py:93).
"""

from __future__ import annotations


def pairwise(a) -> float:
    n = len(a)
    if n < 8:
        r = 0.0
        for v in a:
            r += float(v)
        return r
    if n <= 128:
        r = [float(v) for v in a[:8]]
        i = 8
        stop = n - (n % 8)
        while i < stop:
            for j in range(8):
                r[j] += float(a[i + j])
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += float(a[i])
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise(a[:n2]) + pairwise(a[n2:])


def reduceat_segment(col) -> float:
    return float(col[0]) + pairwise(col[1:]) if len(col) > 1 else float(col[0])


def einsum_sq(c) -> float:
    n = len(c)
    a0 = a1 = 0.0
    i = 0
    while n - i >= 8:
        b3_0 = float(c[i + 6]) * float(c[i + 6]) + a0
        b3_1 = float(c[i + 7]) * float(c[i + 7]) + a1
        b2_0 = float(c[i + 4]) * float(c[i + 4]) + b3_0
        b2_1 = float(c[i + 5]) * float(c[i + 5]) + b3_1
        b1_0 = float(c[i + 2]) * float(c[i + 2]) + b2_0
        b1_1 = float(c[i + 3]) * float(c[i + 3]) + b2_1
        a0 = float(c[i]) * float(c[i]) + b1_0
        a1 = float(c[i + 1]) * float(c[i + 1]) + b1_1
        i += 8
    while i < n:
        a0 = float(c[i]) * float(c[i]) + a0
        a1 = (float(c[i + 1]) * float(c[i + 1]) + a1) if i + 1 < n else (0.0 + a1)
        i += 2
    return 0.0 + (a0 + a1)
