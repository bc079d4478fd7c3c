"""World-size-2 gloo test of the distributed control plane (CPU only): the
shared-memory ring delivers every transaction to every worker in order
(transport.py:242-261 dispatch order), survives wrap-around with
back-pressure, and cancel words / result slots written by one process are
seen by the other."""

import os
import struct

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_11798_b200 import dist as D
from paper_2407_11798_b200.model import TOKEN_DTYPE

N_REC = D.RING * 2 + 37     # force wrap-around


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    name = ["sp_test_%d" % port if rank == 0 else None]
    dist.broadcast_object_list(name, src=0)
    plane = D.ControlPlane(name[0], rank == 0, world, 16, 1) if rank == 0 else None
    dist.barrier()
    if rank != 0:
        plane = D.ControlPlane(name[0], False, world, 16, 1)
    dist.barrier()
    try:
        if rank == 0:
            for i in range(N_REC):
                toks = np.zeros(1 + i % 4, dtype=TOKEN_DTYPE)
                toks["token"] = i
                toks["pos"] = np.arange(len(toks)) + i
                if i % 3 == 0:
                    plane.write(D.R_RUN, D._pack_run(i, 2, 3, toks, list(range(len(toks)))))
                elif i % 3 == 1:
                    plane.write(D.R_COPY, struct.pack("<iIi", i % 8, 0b1010, i))
                else:
                    plane.write(D.R_REMOVE, struct.pack("<ii", i % 8, i))
            plane.cancel[7] = 4103
            plane.write(D.R_SHUTDOWN, b"")
            # wait for the worker's result slot
            while plane.flags[5] != 99:
                pass
            q.put(("r0", int(plane.res[5][0]), int(plane.res[5][4])))
        else:
            seen = []
            while True:
                rtype, p = plane.read(rank)
                if rtype == D.R_SHUTDOWN:
                    break
                if rtype == D.R_RUN:
                    run_id, kind, flags, toks, rows = D._unpack_run(p)
                    ok = (toks["token"] == run_id).all() and list(rows) == list(range(len(toks)))
                    seen.append(("run", run_id, bool(ok)))
                elif rtype == D.R_COPY:
                    seen.append(("copy",) + struct.unpack("<iIi", p[:12]))
                else:
                    seen.append(("remove",) + struct.unpack("<ii", p[:8]))
            plane.res[5][0] = 1
            plane.res[5][4] = 42
            plane.flags[5] = 99
            q.put(("r1", seen, int(plane.cancel[7])))
    finally:
        dist.barrier()
        plane.close(unlink=(rank == 0))
        dist.destroy_process_group()


def test_control_plane_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 200
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((m[0], m[1:]) for m in (q.get(timeout=120), q.get(timeout=120)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    seen, cancel = out["r1"]
    assert len(seen) == N_REC
    for i, s in enumerate(seen):
        if i % 3 == 0:
            assert s == ("run", i, True)
        elif i % 3 == 1:
            assert s == ("copy", i % 8, 0b1010, i)
        else:
            assert s == ("remove", i % 8, i)
    assert cancel == 4103
    assert out["r0"] == (1, 42)


def test_run_record_roundtrip():
    toks = np.zeros(5, dtype=TOKEN_DTYPE)
    toks["token"] = [3, 1, 4, 1, 5]
    toks["pos"] = [9, 10, 11, 12, 13]
    toks["seq_mask"] = 1 << 3
    toks["want_logits"] = 1
    run_id, kind, flags, t2, rows = D._unpack_run(D._pack_run(17, 2, 3, toks, [0, 2, 4]))
    assert (run_id, kind, flags) == (17, 2, 3)
    assert (t2 == toks).all() and list(rows) == [0, 2, 4]


# ---------------------------------------------------------------------------
# The head side of the dedicated-draft layout (rank 0 hosts no stage) over a
# fake last stage on rank 1: RUN records in order, results back through the
# shared result slots (FIFO), COMPACT records every capacity/2 appended
# cells, RESET clears the flags (CPU only: the stage is simulated).
# ---------------------------------------------------------------------------
def _dedicated_worker(rank, world, port, q):
    import time
    from paper_2407_11798_b200 import _lib
    from paper_2407_11798_b200.runtime import RES_DTYPE
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    name = ["sp_test_ded_%d" % port if rank == 0 else None]
    dist.broadcast_object_list(name, src=0)
    plane = D.ControlPlane(name[0], rank == 0, world, 16, 1) if rank == 0 else None
    dist.barrier()
    if rank != 0:
        plane = D.ControlPlane(name[0], False, world, 16, 1)
    dist.barrier()
    try:
        if rank == 0:
            pipe = D.DistPipeline(None, [(0, 4)], plane, world, capacity=64, max_tokens=16,
                                  local_stage=False)
            assert pipe.n_stages == 1 and pipe.stages == []
            got = []
            for rid in range(1, 41):
                toks = np.zeros(3, dtype=TOKEN_DTYPE)
                toks["token"] = rid
                pipe.launch(rid, 2, toks, 0, [0, 2])
                if rid % 4 == 0:
                    while pipe.in_flight():
                        r = pipe.wait()
                        got.append((r.run_id, r.placeholder, [x.argmax for x in r.rows]))
            q.put(("r0", got, pipe.compactions))
            pipe.reset()
            pipe.shutdown()
        else:
            records = []
            while True:
                rtype, p = plane.read(rank)
                records.append(rtype)
                if rtype == D.R_SHUTDOWN:
                    break
                if rtype == D.R_RUN:
                    run_id, kind, flags, toks, rows = D._unpack_run(p)
                    slot = run_id % D.RESULTS
                    blk = plane.res[slot]
                    blk[0] = _lib.SP_STATUS_PLACEHOLDER if run_id % 7 == 0 else _lib.SP_STATUS_VALID
                    blk[1] = 0
                    rr = blk[4:4 + 4 * len(rows)].view(RES_DTYPE)
                    for j, row in enumerate(rows):
                        rr[j]["a"] = 100 * run_id + int(row)
                    plane.flags[slot] = run_id
            q.put(("r1", records))
    finally:
        dist.barrier()
        plane.close(unlink=(rank == 0))
        dist.destroy_process_group()


def test_dedicated_layout_head_side():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29800 + os.getpid() % 150
    procs = [ctx.Process(target=_dedicated_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((m[0], m[1:]) for m in (q.get(timeout=120), q.get(timeout=120)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got, compactions = out["r0"]
    (records,) = out["r1"]
    assert [g[0] for g in got] == list(range(1, 41))          # FIFO
    for rid, ph, rows in got:
        assert ph == (rid % 7 == 0)
        assert rows == ([] if ph else [100 * rid, 100 * rid + 2])
    # 40 runs x 3 cells, compaction every capacity/2 = 32 cells -> 3
    assert compactions == 3 and records.count(D.R_COMPACT) == 3
    assert records.count(D.R_RUN) == 40 and D.R_RESET in records
