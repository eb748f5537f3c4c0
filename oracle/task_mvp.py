"""Task-parallel form of the reference product -- BENCH/TEST INFRASTRUCTURE ONLY.

Restates the reference's dependency-aware task engine
(/root/reference/pkg/src/taskfmm/runtime.py:1-290) and its task submission of
the product (fastmvp.py:62-139, ``mvp`` with a ``Runtime``), so that the
reference's own task-parallel timing can be measured on the GPU box, where
/root/reference does not exist ("mvp with
Runtime(RuntimeConfig(workers=os.cpu_count()))").  Only bench.py's
``--impl reference`` leg and tests/ use it; the product never does.

Semantics kept from runtime.py:
* a handle keeps a queue of generations; consecutive READ or consecutive
  ADD accesses share a generation, anything else starts a new one; only the
  front generation is enabled, a task is ready when all its accesses are
  (runtime.py:137-161, 262-276);
* ADD accesses are mutually exclusive per handle, locks taken in handle-id
  order (runtime.py:219-237);
* every worker owns a FIFO deque, the submitter pushes ready tasks
  round-robin, idle workers steal from the back of other deques
  (runtime.py:190-216).
Tracing and conflict instrumentation are left out (they only observe).
"""

from __future__ import annotations

import itertools
import threading
from collections import deque

import numpy as np

READ, ADD, WRITE = "read", "add", "write"


class Handle:
    __slots__ = ("id", "gens", "lock")

    def __init__(self, hid: int):
        self.id = hid
        self.gens = deque()          # [mode, tasks, completed]
        self.lock = threading.Lock()


class Task:
    __slots__ = ("kind", "accesses", "body", "pending")

    def __init__(self, kind, accesses, body):
        self.kind = kind
        self.accesses = accesses
        self.body = body
        self.pending = 0


class TaskRuntime:
    """Worker threads executing submitted tasks in dependency order."""

    def __init__(self, workers: int):
        self.lock = threading.Lock()
        self.work = threading.Condition(self.lock)
        self.done = threading.Condition(self.lock)
        self.queues = [deque() for _ in range(workers)]
        self.ids = itertools.count()
        self.submitted = self.completed = 0
        self.rr = 0
        self.stop = False
        self.errors = []
        self.threads = [threading.Thread(target=self._worker, args=(w,), daemon=True)
                        for w in range(workers)]
        for t in self.threads:
            t.start()

    def handle(self) -> Handle:
        return Handle(next(self.ids))

    def submit(self, task: Task) -> None:
        with self.lock:
            self.submitted += 1
            pending = 0
            for h, mode in task.accesses:
                g = h.gens
                if g and g[-1][0] == mode and mode in (READ, ADD):
                    gen = g[-1]
                else:
                    gen = [mode, [], 0]
                    g.append(gen)
                gen[1].append(task)
                if gen is not g[0]:
                    pending += 1
            task.pending = pending
            if pending == 0:
                self._push(task)

    def barrier(self) -> None:
        with self.lock:
            while self.completed < self.submitted:
                self.done.wait()
            if self.errors:
                raise self.errors[0]

    def shutdown(self) -> None:
        with self.lock:
            self.stop = True
            self.work.notify_all()
        for t in self.threads:
            t.join()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.shutdown()

    def _push(self, task: Task) -> None:
        self.queues[self.rr].append(task)
        self.rr = (self.rr + 1) % len(self.queues)
        self.work.notify()

    def _take(self, w: int):
        own = self.queues[w]
        if own:
            return own.popleft()
        for v, q in enumerate(self.queues):
            if v != w and q:
                return q.pop()
        return None

    def _worker(self, w: int) -> None:
        while True:
            with self.lock:
                task = self._take(w)
                while task is None and not self.stop:
                    self.work.wait()
                    task = self._take(w)
                if task is None:
                    return
            adds = sorted((h for h, m in task.accesses if m == ADD), key=lambda h: h.id)
            for h in adds:
                h.lock.acquire()
            try:
                task.body()
            except Exception as exc:      # keep the worker alive, re-raise at barrier
                with self.lock:
                    self.errors.append(exc)
            finally:
                for h in reversed(adds):
                    h.lock.release()
                self._complete(task)

    def _complete(self, task: Task) -> None:
        with self.lock:
            for h, _ in task.accesses:
                gen = h.gens[0]
                gen[2] += 1
                if gen[2] == len(gen[1]):
                    h.gens.popleft()
                    if h.gens:
                        for succ in h.gens[0][1]:
                            succ.pending -= 1
                            if succ.pending == 0:
                                self._push(succ)
            self.completed += 1
            if self.completed == self.submitted:
                self.done.notify_all()


def _gemv(A, x, y):
    def run():
        np.add(y, A @ x, out=y)
    return run


def mvp_tasks(tree, ops, q, rt: TaskRuntime, near: bool = True, far: bool = True):
    """phi = K~ q as one task per gemv (fastmvp.py:62-139), real float64 q."""
    q = np.asarray(q, dtype=np.float64)
    if q.shape != (tree.n_points,):
        raise ValueError("q must have one charge per point")
    groups = tree.groups
    G = len(groups)
    Q = ops.params.Q
    leaves = tree.leaves()
    qt = q[tree.perm]
    phi = np.zeros(tree.n_points)
    s = np.zeros((G, Q))
    o = np.zeros((G, Q))
    hq = {g.id: rt.handle() for g in leaves}
    hphi = {g.id: rt.handle() for g in leaves}
    hs = [rt.handle() for _ in range(G)]
    ho = [rt.handle() for _ in range(G)]
    sub = rt.submit
    if near:   # fastmvp.py:68-79
        for a in leaves:
            pa = phi[a.start:a.stop]
            for bid in a.neighbors:
                b = groups[bid]
                sub(Task("near", [(hq[bid], READ), (hphi[a.id], ADD)],
                         _gemv(ops.near[(a.id, bid)], qt[b.start:b.stop], pa)))
    if far:    # fastmvp.py:82-121
        for b in leaves:
            sub(Task("radiation", [(hq[b.id], READ), (hs[b.id], ADD)],
                     _gemv(ops.V[b.id], qt[b.start:b.stop], s[b.id])))
        for level in range(tree.L, tree.l0, -1):
            for gid in tree.level_ids[level]:
                p = groups[gid].parent
                sub(Task("source-transfer", [(hs[gid], READ), (hs[p], ADD)],
                         _gemv(ops.C[gid], s[gid], s[p])))
        for level in range(tree.l0, tree.L + 1):
            for aid in tree.level_ids[level]:
                for bid in groups[aid].interaction:
                    sub(Task("translation", [(hs[bid], READ), (ho[aid], ADD)],
                             _gemv(ops.D[(aid, bid)], s[bid], o[aid])))
        for level in range(tree.l0 + 1, tree.L + 1):
            for gid in tree.level_ids[level]:
                p = groups[gid].parent
                sub(Task("potential-transfer", [(ho[p], READ), (ho[gid], ADD)],
                         _gemv(ops.B[gid], o[p], o[gid])))
        for a in leaves:
            sub(Task("reception", [(ho[a.id], READ), (hphi[a.id], ADD)],
                     _gemv(ops.U[a.id], o[a.id], phi[a.start:a.stop])))
    rt.barrier()
    return phi[tree.inverse_perm()]
