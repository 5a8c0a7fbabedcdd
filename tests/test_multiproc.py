"""N > 1 host logic on CPU: two `gloo` ranks run the C5 batch sharding of
bench.py (`--config c5b`) -- member split, per-rank value sets on the shared
structure, max-over-ranks timing -- with the CPU oracle standing in for the
device factorization (test-only; the product path has no CPU fallback)."""
import os
import socket
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, nmembers, out_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    import torch.distributed as dist

    from checkers import Oracle
    from paper_1601_05871_b200 import batch

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    mine = batch.shard(nmembers, rank, world)
    an, vals, perms = batch.member_values(list(mine))
    O = Oracle()
    hashes = {}
    for m, ap, v in zip(mine, perms, vals):
        ref, st, _, _ = O.factor_serial(ap, an.pattern.pattern)
        assert st == 0
        hashes[m] = O.hash(ref)
    gathered = [None] * world
    dist.all_gather_object(gathered, (list(mine), hashes))
    t = batch.max_over_ranks(1.0 + rank)
    if rank == 0:
        with open(os.path.join(out_dir, "result.txt"), "w") as f:
            f.write(repr((gathered, t)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("nmembers", [5])
def test_two_rank_c5_batch_sharding(tmp_path, nmembers):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(worker, args=(world, free_port(), nmembers, str(tmp_path)), nprocs=world, join=True)
    gathered, t = eval(open(tmp_path / "result.txt").read())
    assert t == 2.0  # max over ranks
    owned = [m for ms, _ in gathered for m in ms]
    assert sorted(owned) == list(range(nmembers))  # disjoint and complete
    assert [len(ms) for ms, _ in gathered] == [3, 2]
    # every rank's factors equal the single-process ones
    sys.path.insert(0, HERE)
    from checkers import Oracle
    from paper_1601_05871_b200 import batch
    an, _, perms = batch.member_values(range(nmembers))
    O = Oracle()
    merged = {m: h for _, hs in gathered for m, h in hs.items()}
    for m, ap in enumerate(perms):
        assert merged[m] == O.hash(O.factor_serial(ap, an.pattern.pattern)[0])


def test_shard_sizes():
    from paper_1601_05871_b200 import batch
    for n, w in [(64, 1), (64, 2), (64, 8), (10, 3), (3, 8)]:
        parts = [batch.shard(n, r, w) for r in range(w)]
        assert sum(len(p) for p in parts) == n
        assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
        assert [x for p in parts for x in p] == list(range(n))
    with pytest.raises(ValueError):
        batch.shard(4, 2, 2)


def shard_worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    import torch.distributed as dist

    from conftest import analyzed, planned
    from test_plan import part_tables

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    # what bench.py run_sharded does per rank before the GPU work
    _, an = analyzed("c5_m0")
    plan = planned("c5_m0")
    owners = an.subtree_owners(world, separators=0)
    mine = part_tables(plan.part_problem(world, owners, rank))
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    if rank == 0:
        np.save(os.path.join(out_dir, "owners.npy"), owners)
        import pickle
        with open(os.path.join(out_dir, "parts.pkl"), "wb") as f:
            pickle.dump(parts, f)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_subtree_sharding(tmp_path, oracle):
    # C6 sharding host side over two gloo ranks: each rank builds its part
    # (rows of its ND subtree, remote operands encoded); rank 0 collects them
    # and the CPU replay of all parts equals factor_serial bit for bit
    import pickle

    import torch.multiprocessing as mp
    sys.path.insert(0, HERE)
    from conftest import analyzed, bitwise_equal, planned
    from test_plan import replay_parts
    mp.spawn(shard_worker, args=(2, free_port(), str(tmp_path)), nprocs=2, join=True)
    owners = np.load(tmp_path / "owners.npy")
    parts = pickle.load(open(tmp_path / "parts.pkl", "rb"))
    assert [int((owners == k).sum()) > 0 for k in range(2)] == [True, True]
    from checkers import flow_programs
    f = planned("c5_m0").flow_tables()
    slot, upd = flow_programs(f["row_ptr"], f["cols"])
    full, remote, read_remotely, exported = replay_parts(f, slot, upd, parts, owners)
    _, an = analyzed("c5_m0")
    ref, _, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    assert bitwise_equal(full, ref) and remote > 0 and read_remotely <= exported


def sharded_run_worker(rank, world, port, out_dir, name, separators):
    """bench.py run_sharded on CPU ranks: phase 1 (reset), barrier, phase 2
    (this rank's rows in its schedule order, operands of other parts read
    from what they published), then the disjoint-row all_reduce assembly.
    The device's peer reads become an exchange after every round: a rank
    publishes only the rows flagged exported (bit 31 of the record), so a
    missing flag would stall the run and fail the test."""
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    import torch
    import torch.distributed as dist

    from checkers import flow_programs
    from conftest import analyzed, planned
    from test_plan import part_programs, part_tables

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    _, an = analyzed(name)
    plan = planned(name)
    owners = an.subtree_owners(world, separators=separators)
    part = part_tables(plan.part_problem(world, owners, rank))
    f = plan.flow_tables()
    slot, upd = flow_programs(f["row_ptr"], f["cols"])
    rowid = np.repeat(np.arange(len(f["row_ptr"]) - 1), np.diff(f["row_ptr"]))
    ps, pu = part_programs(slot, upd, rowid, owners, rank)
    a = f["values"]
    # phase 1: this part's U <- unwritten, on every rank before any row runs
    out = np.full(len(a), np.nan)
    done = np.zeros(len(a), bool)
    dist.barrier()
    # phase 2
    remote = {}  # (owner, position) -> published value
    nxt, rounds, stalls = 0, 0, 0
    rows = len(part["rec"])

    def operand(x):
        if x & 0x80000000:
            key = ((x >> 25) & 63, x & 0x1FFFFFF)
            return remote.get(key)
        return out[x] if done[x] else None

    while True:
        outbox, progressed = [], 0
        while nxt < rows:
            tb, lk, dpos, _ = (int(x) for x in part["rec"][nxt])
            L, kind = lk & ((1 << 30) - 1), (lk >> 30) & 1
            v = a[tb:tb + L].copy()
            ready = kind == 0 or done[dpos]
            for j in range(L):
                for m, o in pu[ps[tb + j, 0]:ps[tb + j, 1]]:
                    x, y = operand(int(m)), operand(int(o))
                    if x is None or y is None:
                        ready = False
                        break
                    v[j] = v[j] - x * y
                if not ready:
                    break
            if not ready:
                break  # in order, like one warp: the next rows wait too
            if kind == 0:
                d = np.sqrt(v[0])
                v[1:] = v[1:] / d
                v[0] = d
            else:
                v = v / out[dpos]
            out[tb:tb + L] = v
            done[tb:tb + L] = True
            if lk < 0:  # exported: other parts read this row
                outbox.extend((rank, tb + j, float(v[j])) for j in range(L))
            nxt += 1
            progressed += 1
        got = [None] * world
        dist.all_gather_object(got, (outbox, progressed, nxt == rows))
        for box, _, _ in got:
            for ow, pos, val in box:
                remote[(ow, pos)] = val
        rounds += 1
        if all(fin for _, _, fin in got):
            break
        stalls = stalls + 1 if sum(p for _, p, _ in got) == 0 else 0
        assert stalls < 2, "sharded schedule stalled"
    # assembly as bench.py: every rank contributes its rows, the sum is the factor
    own = np.repeat(owners, np.diff(f["row_ptr"])) == rank
    mine = torch.from_numpy(np.where(own, out, 0.0))
    dist.all_reduce(mine)
    if rank == 0:
        np.save(os.path.join(out_dir, "factor.npy"), mine.numpy())
        with open(os.path.join(out_dir, "rounds.txt"), "w") as fh:
            fh.write(str(rounds))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world,separators", [("c5_m0", 2, "spread"), ("c1", 4, "spread"),
                                                   ("c5_m0", 2, 0)])
def test_sharded_run_phases_and_exchange(tmp_path, oracle, name, world, separators):
    # run_sharded's protocol across gloo ranks, each with its own copy of U:
    # bitwise equal to factor_serial, no stall, separators spread or on rank 0
    import torch.multiprocessing as mp
    sys.path.insert(0, HERE)
    from conftest import analyzed, bitwise_equal
    mp.spawn(sharded_run_worker, args=(world, free_port(), str(tmp_path), name, separators), nprocs=world,
             join=True)
    got = np.load(tmp_path / "factor.npy")
    _, an = analyzed(name)
    ref, _, _, _ = oracle.factor_serial(an.a_permuted, an.pattern.pattern)
    assert bitwise_equal(got, ref)
    assert int(open(tmp_path / "rounds.txt").read()) > 1


def test_spread_separators_one_per_part():
    sys.path.insert(0, HERE)
    from conftest import analyzed
    _, an = analyzed("c2")
    for world in (2, 4, 8):
        base = an.subtree_owners(world)
        spread = an.subtree_owners(world, separators="spread")
        lo, hi = an.subtree_spans[world.bit_length() - 1]
        inside = np.zeros(len(base), bool)
        for a, b in zip(lo, hi):
            inside[a:b] = True
        assert np.array_equal(base[inside], spread[inside])  # subtrees unchanged
        moved = np.unique(spread[~inside])
        assert len(moved) == min(world - 1, world)  # N-1 separators, each on its own part
