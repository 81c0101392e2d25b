"""CPU-side checks of the C ABI (no GPU needed): the library loads, exports
every function include/pbicgstab.h declares, and its host-only logic
(partition, halo plan, superaccumulator merge+round twin) is right, including
a world_size-2 gloo run of the cross-rank superaccumulator reduction."""
import os
import re
import struct

import numpy as np
import pytest

import gen
import oracle
import paper_2404_13216_b200 as pb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bits(v):
    return struct.unpack("<Q", struct.pack("<d", v))[0]


def header_functions():
    src = open(os.path.join(ROOT, "include", "pbicgstab.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|void|const char \*)\s*\*?\s*(\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_header_symbol():
    L = pb.lib()
    names = header_functions()
    assert len(names) >= 15, names
    for nm in names:
        assert hasattr(L, nm), nm
    assert L.pbcg_abi_version() == 10


def test_plan_partition_spec_examples():
    # SPEC.md l.185-187
    assert list(pb.plan_partition(10, 1)) == [0, 10]
    assert list(np.diff(pb.plan_partition(10, 3))) == [4, 3, 3]
    b = pb.plan_partition(1138, 16)
    assert b[0] == 0 and b[-1] == 1138 and set(np.diff(b)) <= {71, 72}


def _ranges(A, P):
    b = pb.plan_partition(A.n, P)
    out = []
    for q in range(P):
        s, e = A.row_ptr[b[q]], A.row_ptr[b[q + 1]]
        c = A.col[s:e]
        out.append([b[q], b[q + 1], c.min() if c.size else 0, c.max() if c.size else -1])
    return np.array(out, np.int64)


@pytest.mark.parametrize("P", [2, 3, 8])
def test_plan_halo_consistent(P):
    for A in (gen.stencil(3, 10, 100.0), gen.random_banded(4000, seed=1, band=300)):
        rg = _ranges(A, P)
        plans = [pb.plan_halo(rg, me) for me in range(P)]
        for me in range(P):
            pm = plans[me]
            assert pm["buf_lo"] <= rg[me, 0] and pm["buf_hi"] >= rg[me, 1]
            assert pm["buf_lo"] <= rg[me, 2] and pm["buf_hi"] > rg[me, 3]
            need = set(range(pm["buf_lo"], pm["buf_hi"])) - set(range(rg[me, 0], rg[me, 1]))
            got = set()
            for q in range(P):
                lo, hi = pm["recv_lo"][q], pm["recv_hi"][q]
                got |= set(range(lo, hi))
                # what q sends to me is exactly what I receive from q
                assert plans[q]["send_lo"][me] == lo and plans[q]["send_hi"][me] == hi
                if hi > lo:
                    assert rg[q, 0] <= lo and hi <= rg[q, 1]
            assert got == need


def test_plan_halo_rejects_non_tiling():
    rg = np.array([[0, 5, 0, 6], [6, 10, 4, 9]], np.int64)
    with pytest.raises(pb.PbcgError):
        pb.plan_halo(rg, 0)


@pytest.mark.parametrize("seed", range(8))
def test_host_superacc_twin_rounds_like_oracle(seed):
    # the library's normalise + round (same source as the device path) on the
    # host, against the oracle's independent big-integer EXDOT
    kinds = [lambda: (gen.uniform(5000, seed), gen.uniform(5000, seed + 50)),
             lambda: gen.ill_pair(4096, seed=seed, block=1024),
             lambda: (gen.loguniform(3000, seed, -150, 150), gen.loguniform(3000, seed + 9, -150, 150))]
    x, y = kinds[seed % 3]()
    want, f = oracle.exdot(x, y)
    assert f == 0
    assert bits(pb.sacc_round(pb.sacc_accumulate(x, y))) == bits(want)


def test_host_superacc_special_values():
    assert bits(pb.sacc_round(pb.sacc_accumulate([], []))) == bits(0.0)
    assert pb.sacc_round(pb.sacc_accumulate([1e16, 1.0, -1e16], [1, 1, 1])) == 1.0
    assert pb.sacc_round(pb.sacc_accumulate([1.0, 2.0 ** -53], [1, 1])) == 1.0
    assert pb.sacc_round(pb.sacc_accumulate([1.0 + 2.0 ** -52, 2.0 ** -53], [1, 1])) == 1.0 + 2.0 ** -51
    u = 2.0 ** -52
    x = [(1 + u) * 2.0 ** -480, -(1 + 2 * u) * 2.0 ** -480]
    y = [(1 + u) * 2.0 ** -480, 2.0 ** -480]
    assert pb.sacc_round(pb.sacc_accumulate(x, y)) == 2.0 ** -1064
    # overflow of the rounded sum: word 66 weighs 2^(32*66-1074) = 2^1038
    w = np.zeros(pb.sacc_words(), np.int64)
    w[-1] = 1
    assert pb.sacc_round(w) == float("inf")
    w[-1] = -1
    assert pb.sacc_round(w) == float("-inf")
    w[:] = 0
    w[-1] = -(1 << 40)  # large negative top word, still exact arithmetic
    assert pb.sacc_round(w) == float("-inf")
    # largest finite: (2 - 2^-52) * 2^1023 deposited exactly
    big = np.nextafter(np.inf, 0)
    assert pb.sacc_round(pb.sacc_accumulate([big], [1.0])) == big
    # subnormal result (words hold multiples of 2^-1074)
    assert pb.sacc_round(pb.sacc_accumulate([2.0 ** -1000, -(2.0 ** -1000)], [2.0 ** 40, 2.0 ** 40 - 2.0 ** -12])) \
        == oracle.exdot([2.0 ** -1000, -(2.0 ** -1000)], [2.0 ** 40, 2.0 ** 40 - 2.0 ** -12])[0]


def _gloo_worker(rank, world, port, x, y, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = pb.plan_partition(x.size, world)
    w = torch.from_numpy(pb.sacc_accumulate(x[b[rank]:b[rank + 1]], y[b[rank]:b[rank + 1]]))
    dist.all_reduce(w, op=dist.ReduceOp.SUM)  # exact, order-independent int64 sum
    r = pb.sacc_round(w.numpy())
    # halo plan agreement across ranks through an allgather of the row ranges
    A = gen.stencil(3, 8, 100.0)
    rb = pb.plan_partition(A.n, world)
    s, e = A.row_ptr[rb[rank]], A.row_ptr[rb[rank + 1]]
    mine = torch.tensor([rb[rank], rb[rank + 1], A.col[s:e].min(), A.col[s:e].max()], dtype=torch.int64)
    allr = [torch.zeros(4, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allr, mine)
    plan = pb.plan_halo(torch.stack(allr).numpy(), rank)
    send = torch.tensor(np.stack([plan["send_lo"], plan["send_hi"]]), dtype=torch.int64)
    sends = [torch.zeros_like(send) for _ in range(world)]
    dist.all_gather(sends, send)
    ok = all(sends[qq][0, rank] == plan["recv_lo"][qq] and sends[qq][1, rank] == plan["recv_hi"][qq]
             for qq in range(world))
    q.put((rank, r, ok))
    dist.destroy_process_group()


def test_gloo_world2_superacc_allreduce_and_halo():
    import multiprocessing as mp
    import socket
    x, y = gen.ill_pair(1 << 13, seed=11, block=1 << 11)
    want = oracle.exdot(x, y)[0]
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, x, y, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, r, ok in out:
        assert bits(r) == bits(want), rank
        assert ok


# ---- collective contract of setup: config hash + rank records ----

def test_config_hash_and_rank_check():
    h = pb.config_hash(1000, nranks=4)
    assert h == pb.config_hash(1000, nranks=4)
    for other in (pb.config_hash(1001, nranks=4), pb.config_hash(1000, nranks=2), pb.config_hash(None, nranks=4),
                  pb.config_hash(1000, nranks=4, precond="jacobi"), pb.config_hash(1000, nranks=4, comm_mode=1)):
        assert other != h
    b = pb.plan_partition(1000, 4)
    rec = [[b[k], b[k + 1], 0, 999, h] for k in range(4)]
    assert pb.check_ranks(rec, 1000)[0] == 0
    bad = [list(r) for r in rec]
    bad[2][4] = pb.config_hash(1000, nranks=4, precond="jacobi")
    rc, msg = pb.check_ranks(bad, 1000)
    assert rc == 1 and "rank 2" in msg
    gap = [list(r) for r in rec]
    gap[1][1] -= 1  # rows [b2 - 1, b2) owned by nobody
    assert pb.check_ranks(gap, 1000)[0] == 1
    assert pb.check_ranks(gap, 1000, has_matrix=False)[0] == 0  # comm-only: rows are not checked
    short = [list(r) for r in rec]
    short[3][1] = 999
    assert pb.check_ranks(short, 1000)[0] == 1


def _gloo_contract_worker(rank, world, port, n_mine, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = pb.plan_partition(1000, world)
    rec = torch.tensor([[int(b[rank]), int(b[rank + 1]), 0, 999,
                         np.uint64(pb.config_hash(n_mine, nranks=world)).view(np.int64)]], dtype=torch.int64)
    outs = [torch.zeros_like(rec) for _ in range(world)]
    dist.all_gather(outs, rec)
    rc, msg = pb.check_ranks(torch.cat(outs).numpy(), 1000)
    q.put((rank, rc))
    dist.destroy_process_group()


@pytest.mark.parametrize("mismatch", [False, True])
def test_gloo_world2_setup_contract(mismatch):
    # the setup check as two processes run it: every rank sees the same
    # gathered records and returns the same code
    import multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ns = [1000, 1001 if mismatch else 1000]
    ps = [ctx.Process(target=_gloo_contract_worker, args=(r, 2, port, ns[r], q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0] == out[1] == (1 if mismatch else 0)


def test_history_digest_host_twin():
    # pbcg_result.digest's definition (include/pbicgstab.h), written out in
    # Python: FNV-1a 64 over the per-row FNV-1a 64 hashes of the rows' bits
    import paper_2404_13216_b200 as pb
    B, P, M = 0xcbf29ce484222325, 0x100000001b3, (1 << 64) - 1

    def ref(H):
        h = B
        for row in np.ascontiguousarray(H, np.float64).reshape(-1, 12).view(np.uint64):
            rh = B
            for w in row:
                rh = ((rh ^ int(w)) * P) & M
            h = ((h ^ rh) * P) & M
        return h

    rng = np.random.default_rng(5)
    H = rng.standard_normal((9, 12))
    H[3, 4] = -0.0
    H[5, :] = np.nan
    assert pb.history_digest(H) == ref(H)
    assert pb.history_digest(np.zeros((0, 12))) == B
    H2 = H.copy()
    H2[8, 11] = np.nextafter(H2[8, 11], 1.0)  # one ulp anywhere changes it
    assert pb.history_digest(H2) != pb.history_digest(H)
    H3 = H.copy()
    H3[3, 4] = 0.0  # and so does the sign of a zero
    assert pb.history_digest(H3) != pb.history_digest(H)
