"""The fused diagonal factor's task schedule (potrf_diag_fused_kernel,
csrc/small_kernels.cu: FdShape and the waits of the ticket loop), restated
here and checked on the CPU for every order it accepts:

* progress: every wait of a task is on tasks with smaller tickets — the
  kernel's deadlock-freedom argument (a ticket is only held by a running
  CTA, and running CTAs only wait on smaller tickets);
* coverage: the update tasks of step j cover every lower 64 x 64 unit right
  of tile column j exactly once, and the TRSM chunks cover the rows below;
* the chunk indices an update waits for lie inside its step's chunks.
A mismatch here would be a hang (bounded in the kernel, but a wrong result)
for some matrix order the GPU tests do not reach."""
from __future__ import annotations

import pytest

B = 128


class Shape:  # FdShape
    def __init__(self, n: int) -> None:
        self.n, self.T, self.NS = n, -(-n // B), -(-n // 64)

    def units(self, x: int) -> int:
        return 2 * self.NS - 4 * x - 1 if 2 * x + 1 < self.NS else self.NS - 2 * x

    def chunks(self, c: int) -> int:
        return (self.n - (c + 1) * B + 31) // 32 if (c + 1) * B < self.n else 0

    def round_size(self, c: int) -> int:
        return 1 + self.chunks(c) + ((c + 1) * self.units(c + 1) if c + 1 < self.T else 0)

    def unit(self, x: int, u: int) -> tuple[int, int]:
        J0 = 2 * x
        if 2 * x + 1 >= self.NS:
            return J0 + u, J0
        if u < 3:
            return J0 + (u > 0), J0 + (u == 2)
        return J0 + 2 + (u - 3) // 2, J0 + (u - 3) % 2


def tasks(sh: Shape):
    """(ticket, kind, args) in ticket order, decoded as the kernel does"""
    t = 0
    for c in range(sh.T):
        U = sh.units(c + 1) if c + 1 < sh.T else 0
        R = sh.chunks(c)
        for q in range(sh.round_size(c)):
            if q == 0:
                yield t, "L", (c,)
            else:
                q1 = q - 1
                if q1 < c * U:
                    yield t, "S", (q1 // U, c + 1, q1 % U)
                elif q1 - c * U < R:
                    yield t, "T", (c, q1 - c * U)
                else:
                    yield t, "S", (c, c + 1, q1 - c * U - R)
            t += 1


def check(n: int) -> None:
    sh = Shape(n)
    leaf, trsm, upd = {}, {}, {}  # task -> ticket
    order = list(tasks(sh))
    for t, kind, a in order:
        if kind == "L":
            leaf[a[0]] = t
        elif kind == "T":
            trsm[a] = t
        else:
            j, x, u = a
            I, J = sh.unit(x, u)
            assert (j, I, J) not in upd, f"n={n}: unit ({I},{J}) twice in step {j}"
            upd[(j, I, J)] = t
    # coverage
    for j in range(sh.T):
        want = {(j, I, J) for J in range(2 * (j + 1), sh.NS) for I in range(J, sh.NS)}
        got = {k for k in upd if k[0] == j}
        assert got == want, f"n={n} step {j}"
        rows = set()
        for r in range(sh.chunks(j)):
            rows.update(range((j + 1) * B + 32 * r, min((j + 1) * B + 32 * r + 32, n)))
        assert rows == set(range((j + 1) * B, n)) if (j + 1) * B < n else not rows
    # progress: every wait on a smaller ticket
    def before(dep_t, t, what):
        assert dep_t < t, f"n={n}: {what} waits on a later ticket"

    for t, kind, a in order:
        if kind == "L":
            c = a[0]
            J0 = 2 * c
            for I, J in ([(J0, J0)] + ([(J0 + 1, J0), (J0 + 1, J0 + 1)] if J0 + 1 < sh.NS else [])):
                for j in range(c):  # ucnt(I, J) >= c
                    before(upd[(j, I, J)], t, f"L({c})")
        elif kind == "T":
            c, r = a
            before(leaf[c], t, f"T({c},{r})")
            I = ((c + 1) * B + 32 * r) // 64
            for J in [2 * c] + ([2 * c + 1] if 2 * c + 1 < sh.NS else []):
                for j in range(c):
                    before(upd[(j, I, J)], t, f"T({c},{r})")
        else:
            j, x, u = a
            I, J = sh.unit(x, u)
            r0, nr = (j + 1) * B, sh.chunks(j)
            ci, cj = (64 * I - r0) // 32, (64 * J - r0) // 32
            waits = {ci, cj} | ({ci + 1} if ci + 1 < nr else set()) | ({cj + 1} if cj + 1 < nr else set())
            for r in waits:
                assert 0 <= r < nr, f"n={n}: chunk {r} of step {j}"
                before(trsm[(j, r)], t, f"S({j},{x},{u})")
            # the chunks hold every row of both operand row blocks
            for blk in (I, J):
                for row in range(64 * blk, min(64 * blk + 64, n)):
                    assert (row - r0) // 32 in waits
            if j > 0:
                before(upd[(j - 1, I, J)], t, f"S({j},{x},{u})")


@pytest.mark.parametrize("n", [129, 130, 191, 192, 193, 255, 256, 257, 300, 383, 384, 385, 448, 449, 511, 512,
                               700, 777, 1000, 1023, 1024, 1025, 1500, 1983, 2000, 2047, 2048])
def test_fused_diag_schedule_progress_and_coverage(n):
    check(n)


def test_fused_diag_schedule_all_orders_sampled():
    for n in range(129, 2049, 7):
        check(n)
