"""TP group host protocol (include/cake/tp.hpp) at world_size 2 on CPU.

The GPU path (gpu_runtime.cpp run_live_gpu / run_follower) drives the same
coordinator: the leader runs the one scheduler and publishes its compute
launches and loader claims; followers mirror them so NCCL collectives pair up
and every rank loads its own KV-head shard. Here two gloo processes play leader
and follower over the C ABI (cake_tp_*), and gloo checks both saw the same
decisions, the landed barrier held, and back-to-back runs reset cleanly.
"""
import ctypes as C
import os
import threading
import uuid

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_03065_b200 import native as N


RACE_BIT = 1 << 30  # include/cake_c.h CAKE_TP_RACE_BIT


def _split(n, run):
    # compute takes the prefix, io the suffix backward (the bidirectional shape);
    # the merge point moves between runs
    m = max(1, n // 2 + (run % 3) - 1)
    return list(range(m)), list(range(n - 1, m - 1, -1))


def _worker(rank, world, port, shm, n, runs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lib = N.load()
        h = N.vp()
        lib.call("cake_tp_create", shm.encode(), rank, world, C.byref(h))
        t = h.value
        seen = []
        for run in range(1, runs + 1):
            lib.call("cake_tp_begin_run", t, run, n)
            comp, io_seq = _split(n, run)
            got_c, got_io, final, raced = [], [], None, []
            if rank == 0:
                def loader():
                    for i in io_seq:
                        lib.call("cake_tp_publish_io", t, i)
                        lib.call("cake_tp_shard_landed", t, i)
                        lib.call("cake_tp_wait_all_landed", t, i)  # commit only when every shard landed
                        got_io.append(i)
                th = threading.Thread(target=loader)
                th.start()
                for i in comp:
                    lib.call("cake_tp_publish_compute", t, i | (RACE_BIT if i == comp[-1] else 0))
                    got_c.append(i)
                lib.call("cake_tp_end_compute", t)
                th.join()
                lib.call("cake_tp_end_io", t)
                # a chunk the compute side committed: waiting for its shards returns at once
                # (the loads were dropped) instead of waiting for shards that never land
                lib.call("cake_tp_publish_decided", t, comp[0], 1)
                lib.call("cake_tp_wait_all_landed", t, comp[0])
                # the contested chunk of this run: compute's last entry raced (kRaceBit), io won it
                lib.call("cake_tp_publish_decided", t, comp[-1], 2)
                lib.call("cake_tp_publish_final", t, run % 2, 17 + run, comp[-1])
                final = (run % 2, 17 + run, comp[-1], 2)
            else:
                def mirror_io():
                    k = 0
                    while True:
                        c, has = N.u32(), C.c_int()
                        lib.call("cake_tp_next_io", t, k, C.byref(c), C.byref(has))
                        if not has.value:
                            break
                        got_io.append(c.value)
                        lib.call("cake_tp_shard_landed", t, c.value)
                        k += 1
                th = threading.Thread(target=mirror_io)
                th.start()
                k = 0
                while True:
                    c, has = N.u32(), C.c_int()
                    lib.call("cake_tp_next_compute", t, k, C.byref(c), C.byref(has))
                    if not has.value:
                        break
                    got_c.append(c.value & ~RACE_BIT)
                    if c.value & RACE_BIT:
                        raced.append(c.value & ~RACE_BIT)
                    k += 1
                rc, row, race, side = C.c_int(), C.c_int(), C.c_int(), C.c_int()
                lib.call("cake_tp_wait_final", t, C.byref(rc), C.byref(row), C.byref(race))
                lib.call("cake_tp_decided", t, race.value, C.byref(side))
                final = (rc.value, row.value, race.value, side.value)
                th.join()
            lib.call("cake_tp_end_run", t)
            if rank == 0:
                raced = [comp[-1]]
            seen.append((got_c, got_io, final, raced))
        everyone = [None] * world
        dist.all_gather_object(everyone, seen)
        lib.call("cake_tp_destroy", t)
        if rank == 0:
            q.put(everyone)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [1, 7, 64])
def test_tp_coordinator_world2(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000) + n
    shm = f"/cake_tp_test_{uuid.uuid4().hex[:12]}"
    runs = 3
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shm, n, runs, q)) for r in range(2)]
    for p in procs:
        p.start()
    everyone = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    leader, follower = everyone
    for run, (lc, li, lf, lr) in enumerate(leader, start=1):
        fc, fi, ff, fr = follower[run - 1]
        assert fr == lr  # the racer's entry carried the race bit
        comp, io_seq = _split(n, run)
        assert lc == comp and fc == comp
        assert li == io_seq and fi == io_seq
        assert lf == ff == (run % 2, 17 + run, comp[-1], 2)
        assert sorted(comp + io_seq) == list(range(n))


def test_tp_bad_rank():
    lib = N.load()
    h = N.vp()
    with pytest.raises(ValueError):
        lib.call("cake_tp_create", b"/cake_tp_bad", 3, 2, C.byref(h))
