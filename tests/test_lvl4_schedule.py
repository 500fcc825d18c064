"""The task order of the level-group kernel k_dst_lvl4 (lvl_dst.cuh), restated
in Python and checked on the host: every task is issued exactly once, task
pairs are what the Z discards assume, and every dependency points to a lower
task index -- the property the kernel's deadlock-freedom argument rests on
(all CTAs co-resident, each running its tasks in increasing order, so the
lowest unfinished task never waits).

The restatement follows `decode` and `task_of` of lvl_dst.cuh line for line;
the dependencies are the producer's waits: a column task of level tile g on
g's row-task counter (all 1024 row tasks of g), a row task of tile g >= 2 on
the column-task counter of g - 2 (its Z slot).
"""

import pytest

K_ROW_TASKS = 1024


def decode(i, nt, nct, kfirst):
    """lvl_dst.cuh decode(): task index -> (kind, level tile, idx); kind 0 row, 1 column."""
    pi, u = i >> 1, i & 1
    nb, nc = K_ROW_TASKS // 2, 4 * nct
    per = nb + nc
    if pi < nb:
        kind, g, pidx = 0, 0, pi
    else:
        p = 1 + (pi - nb) // per
        j = pi - nb - (p - 1) * per
        kf = min(kfirst, nb)
        if p >= nt:
            kind, g, pidx = 1, nt - 1, j
        elif j < kf:
            kind, g, pidx = 0, p, j
        elif j < kf + nc:
            kind, g, pidx = 1, p - 1, j - kf
        else:
            kind, g, pidx = 0, p, j - nc
    return kind, g, 2 * pidx + u


def task_of(c, G, it):
    return 2 * c + 2 * G * (it >> 1) + (it & 1)


def ntasks(nlev, nct):
    nt = (nlev + 7) // 8
    return nt * K_ROW_TASKS + nlev * nct


@pytest.mark.parametrize("nlev,grid,kfirst", [(1, 148, 148), (9, 148, 148), (23, 148, 74), (1025, 148, 148),
                                              (1025, 148, 0), (64, 7, 300), (17, 1, 5)])
def test_lvl4_schedule_covers_tasks_and_orders_dependencies(nlev, grid, kfirst):
    nct = 128                        # column tiles per level (m = 1023)
    nt = (nlev + 7) // 8
    n = ntasks(nlev, nct)
    seen = {}
    for i in range(n):
        kind, g, idx = decode(i, nt, nct, kfirst)
        assert 0 <= g < nt
        if kind == 0:
            assert 0 <= idx < K_ROW_TASKS
        else:
            lev = idx // nct
            assert 0 <= lev < 8 and g * 8 + lev < nlev, "a column task of a level past nlev"
        key = (kind, g, idx)
        assert key not in seen, f"task {key} issued twice"
        seen[key] = i
    expected = nt * K_ROW_TASKS + nlev * nct
    assert len(seen) == expected
    # pairs (2i, 2i + 1): same kind and tile; column pairs are the even / odd tile of one
    # 128-byte Z column pair of one level (the odd one discards both)
    for i in range(0, n - 1, 2):
        a, b = decode(i, nt, nct, kfirst), decode(i + 1, nt, nct, kfirst)
        assert a[:2] == b[:2]
        if a[0] == 1:
            assert a[2] // nct == b[2] // nct and a[2] % 2 == 0 and b[2] == a[2] + 1
    # dependencies point to lower task indices
    last_row = {g: max(seen[(0, g, k)] for k in range(K_ROW_TASKS)) for g in range(nt)}
    last_col = {}
    for (kind, g, idx), i in seen.items():
        if kind == 1:
            last_col[g] = max(last_col.get(g, -1), i)
    for (kind, g, idx), i in seen.items():
        if kind == 1:
            assert last_row[g] < i, "a column task before a row task of its level tile"
        elif g >= 2:
            assert last_col[g - 2] < i, "a row task reuses a Z slot before its column tasks"
    # every CTA's slots run in increasing task order and cover every task once
    slots = []
    for c in range(grid):
        prev = -1
        it = 0
        while task_of(c, grid, it) < n:
            t = task_of(c, grid, it)
            assert t > prev
            prev = t
            slots.append(t)
            it += 1
        assert it == ntiles_cta(c, grid, n), "the kernel's closed-form slot count"
    assert sorted(slots) == list(range(n))


def ntiles_cta(c, G, n):
    """k_dst_lvl4's per-CTA slot count (lvl_dst.cuh, before the role split)."""
    c2 = 2 * c
    if n <= c2:
        return 0
    full_pairs = (n - c2) // (2 * G)
    rem = (n - c2) - full_pairs * 2 * G
    return 2 * full_pairs + min(rem, 2)
