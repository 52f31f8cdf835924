"""Concurrent requests on one B200 (the multi-request mix).

The reference serves one request per process (proj/SPEC.md:412 lists fleets as
a non-goal); its bidirectional run (proj/src/scheduler.cpp:229-278) is the unit
this server multiplexes. Design:

* `workers` GpuContexts on one device. The first owns the weights; the others
  share them (cake_model_create_shared) and own their paged KV pool, scratch
  and streams, so each request is a complete bidirectional run (claims,
  loader, race-to-finish, first token) on its own context, and the GPU
  interleaves the contexts' kernels.
* ONE emulated cache-tier link (cake_link / SharedLink): every loader slice of
  every context reserves the next slot of one budget clock, so the requests in
  flight share the link's bandwidth instead of each getting all of it; a
  bandwidth step in the link's trace hits every request at the same instant.
* Requests are dispatched first-come-first-served to the first free context at
  or after their arrival. A request's TTFT is arrival -> first-token logits in
  host memory (queueing included).

Each run's merge point adapts to the bandwidth it actually gets: a request
sharing the link with another sees half the rate, so its compute side takes a
larger share of the prompt.
"""
from __future__ import annotations

import threading
import time
from dataclasses import dataclass, field

from .cake import BandwidthTrace, ChunkStore
from .runtime import GpuResult, GpuRuntime, Link


@dataclass
class Request:
    tier: ChunkStore
    total_tokens: int
    chunk_size: int
    prompt_seed: int
    arrival_ms: float = 0.0
    mode: str = "cake"
    options: dict = field(default_factory=dict)  # GpuRuntime.run keyword options


@dataclass
class Served:
    index: int
    worker: int
    arrival_ms: float   # server clock (t = 0 at serve())
    start_ms: float     # run start on its context
    end_ms: float       # first-token logits in host memory
    ttft_ms: float      # end - arrival
    result: GpuResult
    logits: object = None


class GpuServer:
    def __init__(self, preset, *, workers: int = 2, trace: BandwidthTrace | None = None, mbps: float | None = None,
                 **runtime_kw):
        if workers < 1:
            raise ValueError("workers must be >= 1")
        self.runtimes = [GpuRuntime(preset, **runtime_kw)]
        for _ in range(workers - 1):
            self.runtimes.append(GpuRuntime(preset, weights_from=self.runtimes[0], **runtime_kw))
        self.trace = trace or BandwidthTrace.constant(mbps)
        self.link = Link(self.trace)
        for rt in self.runtimes:
            rt.attach_link(self.link)

    @property
    def primary(self) -> GpuRuntime:
        return self.runtimes[0]

    def serve(self, requests: list[Request], keep_logits: bool = False, after=None) -> list[Served]:
        """Run every request; returns one Served per request (input order).
        after(served, runtime), if given, runs on the worker right after each
        request, before its context takes the next one (e.g. to read its cache)."""
        order = sorted(range(len(requests)), key=lambda i: requests[i].arrival_ms)
        out: list[Served | None] = [None] * len(requests)
        lock = threading.Lock()
        cursor = [0]
        errors: list[BaseException] = []
        self.link.reset()
        t0 = time.perf_counter()

        def now_ms():
            return (time.perf_counter() - t0) * 1e3

        def worker(w: int):
            rt = self.runtimes[w]
            while True:
                with lock:
                    if cursor[0] >= len(order) or errors:
                        return
                    i = order[cursor[0]]
                    cursor[0] += 1
                rq = requests[i]
                wait = rq.arrival_ms - now_ms()
                if wait > 0:
                    time.sleep(wait / 1e3)
                start = now_ms()
                try:
                    r = rt.run(rq.tier, rq.total_tokens, rq.chunk_size, rq.prompt_seed, trace=self.trace,
                               mode=rq.mode, **rq.options)
                except BaseException as e:  # surfaced after the join
                    with lock:
                        errors.append(e)
                    return
                end = start + r.first_token_ms
                out[i] = Served(i, w, rq.arrival_ms, start, end, end - rq.arrival_ms, r,
                                rt.logits() if keep_logits else None)
                if after is not None:
                    try:
                        after(out[i], rt)
                    except BaseException as e:
                        with lock:
                            errors.append(e)
                        return

        threads = [threading.Thread(target=worker, args=(w,), daemon=True) for w in range(len(self.runtimes))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        return out  # type: ignore[return-value]

    def close(self):
        for rt in reversed(self.runtimes):  # siblings before the weight owner
            rt.attach_link(None)
            rt.close()
        self.link.close()
