"""Intra-stage orchestration of several hTasks under tensor parallelism
(paper §3.4.2 "Intra-Stage Orchestration",
P:700-746, Alg. 1 "Priority-Based Subgraph Scheduling").

Several hybrid tasks (hTasks: groups of spatially multiplexed tasks, each one
packed batch and one fused mux_linear call per layer) share a TP group.  The
computation of one hTask overlaps the collectives of another (temporal
multiplexing):

1. Dependency-aware graph construction.  Each hTask's step is an
   ordered list of operators, compute or communication, with the values each
   reads and writes.  Consecutive compute operators cluster into one
   subgraph; each communication operator is appended to the subgraph of the
   operator it depends on.  A new subgraph starts where a compute operator
   reads a value produced by a communication operator of the current one
   (that is the only place execution must wait).  Subgraph priority =
   topological depth.  (The paper isolates small adapters as independent
   subgraphs; here the adapters are fused into the backbone kernel, so there
   is nothing to isolate — DESIGN.md reading R18.)
2. Scheduling (Alg. 1).  A priority queue holds the zero-in-degree subgraphs
   of every DAG; each iteration dequeues the highest-priority one (lowest
   depth, reading R19), among those the longest cumulative compute latency
   ("to maximize overlap with in-flight communication"), ties by
   hTask index; it is recorded with the running timer t and t += latency.
3. Launch (`run_schedule`).  Subgraphs run in schedule order on the caller's
   stream; their trailing collectives are issued asynchronously
   (`async_op=True`: NCCL runs them on its own stream, in issue order, so a
   collective may consume another's output without a wait), and a compute
   operator waits only for the collective handles of the values it reads.
   So hTask i+1's GEMMs run while hTask i's all-gather/reduce-scatter is on
   the wire.  NCCL's CTA budget for the overlapped collectives is capped with
   NCCL_MAX_CTAS (P:791-796 uses 8 CTAs with NVLink SHARP); set by the caller
   before the process group is created (`bench.py --mode tp --comm-ctas`).

Host-side logic only: every arithmetic step is a libmux kernel (or, in the
CPU tests, the injected oracle backend).
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import torch.distributed as dist


@dataclass
class Op:
    """One operator of an hTask's step.  `fn(env)` reads env[v] for v in
    `reads` and stores its outputs into env; a comm op returns a list of
    async work handles (or [] if it completed synchronously)."""
    name: str
    kind: str                      # "compute" | "comm"
    reads: Tuple[str, ...]
    writes: Tuple[str, ...]
    fn: Callable[[dict], Optional[list]]
    latency: float = 0.0           # modeled compute latency (any unit), compute ops only


@dataclass
class Subgraph:
    htask: int
    index: int                     # position within its hTask's DAG
    ops: List[Op]
    deps: List[int] = field(default_factory=list)   # indices (same hTask) it waits on
    depth: int = 0

    @property
    def latency(self) -> float:
        return sum(o.latency for o in self.ops if o.kind == "compute")

    @property
    def key(self) -> Tuple[int, int]:
        return (self.htask, self.index)


def build_subgraphs(htask: int, ops: Sequence[Op]) -> List[Subgraph]:
    """Dependency-aware segmentation of one hTask's operator list."""
    sgs: List[Subgraph] = []
    produced_by: Dict[str, int] = {}        # value -> subgraph index whose comm op writes it
    comm_vals_cur: set = set()
    cur: Optional[Subgraph] = None
    for op in ops:
        if op.kind not in ("compute", "comm"):
            raise ValueError(f"op {op.name}: kind must be compute or comm")
        if cur is None:
            cur = Subgraph(htask, 0, [])
        elif op.kind == "compute" and any(v in comm_vals_cur for v in op.reads):
            sgs.append(cur)
            cur = Subgraph(htask, len(sgs), [])
            comm_vals_cur = set()
        cur.ops.append(op)
        if op.kind == "comm":
            for v in op.writes:
                produced_by[v] = cur.index
                comm_vals_cur.add(v)
    if cur is not None and cur.ops:
        sgs.append(cur)
    # edges: a subgraph depends on every earlier subgraph whose comm output it reads,
    # and (program order within one hTask) on its predecessor
    for sg in sgs:
        deps = set()
        if sg.index > 0:
            deps.add(sg.index - 1)
        for op in sg.ops:
            for v in op.reads:
                j = produced_by.get(v)
                if j is not None and j < sg.index:
                    deps.add(j)
        sg.deps = sorted(deps)
        sg.depth = 0 if not sg.deps else 1 + max(sgs[j].depth for j in sg.deps)
    return sgs


def subgraph_schedule(dags: Sequence[Sequence[Subgraph]]) -> List[Tuple[Subgraph, float]]:
    """Alg. 1: multi-DAG Kahn scheduling, highest priority (lowest depth) first,
    longest cumulative latency among equals.  Returns [(subgraph, t_start)]."""
    indeg: Dict[Tuple[int, int], int] = {}
    children: Dict[Tuple[int, int], List[Subgraph]] = {}
    pq: list = []

    def enqueue(sg: Subgraph):
        heapq.heappush(pq, (sg.depth, -sg.latency, sg.htask, sg.index, sg))

    for dag in dags:
        for sg in dag:
            indeg[sg.key] = len(sg.deps)
            for j in sg.deps:
                children.setdefault((sg.htask, j), []).append(sg)
        for sg in dag:                       # line 3-5: zero in-degree subgraphs
            if indeg[sg.key] == 0:
                enqueue(sg)
    schedule: List[Tuple[Subgraph, float]] = []
    t = 0.0
    while pq:                                # line 6-13
        *_, sg = heapq.heappop(pq)
        for ch in children.get(sg.key, []):
            indeg[ch.key] -= 1
            if indeg[ch.key] == 0:
                enqueue(ch)
        schedule.append((sg, t))
        t += sg.latency
    n = sum(len(d) for d in dags)
    if len(schedule) != n:
        raise ValueError("subgraph dependencies contain a cycle")
    return schedule


def run_schedule(schedule: Sequence[Tuple[Subgraph, float]], envs: Sequence[dict]) -> None:
    """Launch the schedule: compute ops in order on the caller's stream, comm
    ops asynchronous; a compute op waits only for the handles of the values it
    reads.  All outstanding collectives are waited for at the end."""
    pending: List[Dict[str, list]] = [dict() for _ in envs]
    for sg, _t in schedule:
        env, pend = envs[sg.htask], pending[sg.htask]
        for op in sg.ops:
            # a collective reading another collective's output is ordered by the
            # process group's own stream; only compute waits (keeps overlap)
            if op.kind == "compute":
                for v in op.reads:
                    works = pend.pop(v, None)
                    if works:
                        for wk in works:
                            wk.wait()
            works = op.fn(env)
            if op.kind == "comm" and works:
                for v in op.writes:
                    pend[v] = list(works)
    for pend in pending:
        for works in pend.values():
            for wk in works:
                wk.wait()


# ------------------------------------------------------------------ async collectives
def _is_nccl(group) -> bool:
    return dist.get_backend(group) == "nccl"


def all_gather_rows_async(x, out, group=None) -> list:
    """out [p*rows, ...] <- AG(x [rows, ...]).  Async on NCCL; synchronous on gloo."""
    p = dist.get_world_size(group)
    if _is_nccl(group):
        return [dist.all_gather_into_tensor(out, x.contiguous(), group=group, async_op=True)]
    parts = list(out.chunk(p, 0))
    dist.all_gather(parts, x.contiguous(), group=group)
    return []


def reduce_scatter_rows_async(x, out, group=None) -> list:
    """out [rows/p, ...] <- RS(x [rows, ...]) (sum)."""
    p, r = dist.get_world_size(group), dist.get_rank(group)
    if _is_nccl(group):
        return [dist.reduce_scatter_tensor(out, x.contiguous(), group=group, async_op=True)]
    y = x.clone()
    dist.all_reduce(y, group=group)
    rows = x.shape[0] // p
    out.copy_(y[r * rows:(r + 1) * rows])
    return []


def all_reduce_async(xs, group=None) -> list:
    works = []
    for x in xs:
        if x is None:
            continue
        if _is_nccl(group):
            works.append(dist.all_reduce(x, group=group, async_op=True))
        else:
            dist.all_reduce(x, group=group)
    return works


# ------------------------------------------------------------------ the TP layer chain as ops
def linear_chain_ops(layers: Sequence, kinds: Sequence[str], seg_off, seg_task, x_rows_fn, dy,
                     flops_per_layer: Sequence[float], group=None) -> List[Op]:
    """Operator list of one hTask's fwd+bwd step through a TP layer chain.

    `layers[i]` is a tp.ColumnParallelMuxLinear ("col") or
    tp.RowParallelMuxLinear ("row") on this rank's shard; `x_rows_fn(env)`
    produces this rank's row block of the chain input (e.g. the Dispatch
    gather); `dy` is the loss gradient in the last layer's output layout.
    Each layer contributes its compute ops (fused fwd / bwd kernel) and the
    collectives tp.py's layer classes perform, in the same order, so the
    result equals the sequential execution of those classes bit for bit."""
    import torch
    ops: List[Op] = []
    L = len(layers)

    def comp(name, reads, writes, fn, lat=0.0):
        ops.append(Op(name, "compute", tuple(reads), tuple(writes), fn, lat))

    def comm(name, reads, writes, fn):
        ops.append(Op(name, "comm", tuple(reads), tuple(writes), fn))

    comp("dispatch", (), ("x_rows",), lambda e: e.__setitem__("x_rows", x_rows_fn(e)))
    cur = "x_rows"
    for i, (lay, kind) in enumerate(zip(layers, kinds)):
        if kind == "col" and getattr(lay, "fused_ag", False):
            # the all-gather is pushed by the copy engines and consumed inside the GEMM
            def fwd(e, i=i, src=cur, lay=lay):
                e[f"Y{i}"], lay.Hs, lay.X = lay.be.fwd_ag(lay, seg_off, seg_task, e[src])
            comp(f"fwd{i}", (cur,), (f"Y{i}",), fwd, flops_per_layer[i])
            cur = f"Y{i}"
        elif kind == "col":
            def ag(e, i=i, src=cur, lay=lay):
                x = e[src]
                p = dist.get_world_size(group)
                out = torch.empty((x.shape[0] * p,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
                e[f"X{i}"] = out
                return all_gather_rows_async(x, out, group)
            comm(f"AG(x{i})", (cur,), (f"X{i}",), ag)

            def fwd(e, i=i, lay=lay):
                lay.X = e[f"X{i}"]
                Y, lay.Hs = lay.be.fwd(seg_off, seg_task, lay.ads, lay.X, lay.W, lay.r_cap)
                e[f"Y{i}"] = Y
            comp(f"fwd{i}", (f"X{i}",), (f"Y{i}",), fwd, flops_per_layer[i])
            cur = f"Y{i}"
        elif kind == "row" and getattr(lay, "fused_rs", False):
            # the reduce-scatter happens inside the GEMM (peer stores) + the owner-side sum
            def fwd(e, i=i, src=cur, lay=lay):
                lay.X = e[src]
                e[f"Y{i}"], lay.Hs = lay.be.fwd_rs(lay, seg_off, seg_task, lay.X)
            comp(f"fwd{i}", (cur,), (f"Y{i}",), fwd, flops_per_layer[i])
            cur = f"Y{i}"
        elif kind == "row":
            def fwd(e, i=i, src=cur, lay=lay):
                lay.X = e[src]
                e[f"Yp{i}"], lay.Hs = lay.be.fwd(seg_off, seg_task, lay.ads, lay.X, lay.W, lay.r_cap)
            comp(f"fwd{i}", (cur,), (f"Yp{i}",), fwd, flops_per_layer[i])

            def rs(e, i=i):
                y = e[f"Yp{i}"]
                p = dist.get_world_size(group)
                out = torch.empty((y.shape[0] // p,) + tuple(y.shape[1:]), dtype=y.dtype, device=y.device)
                e[f"Y{i}"] = out
                return reduce_scatter_rows_async(y, out, group)
            comm(f"RS(y{i})", (f"Yp{i}",), (f"Y{i}",), rs)
            cur = f"Y{i}"
        else:
            raise ValueError(kind)
    ops.append(Op("loss_grad", "compute", (cur,), (f"dY{L - 1}",),
                  lambda e: e.__setitem__(f"dY{L - 1}", dy)))
    g = f"dY{L - 1}"
    for i in reversed(range(L)):
        lay, kind = layers[i], kinds[i]
        if kind == "col" and getattr(lay, "fused_rs", False):
            def bwd(e, i=i, src=g, lay=lay):
                e[f"dX{i}"], e[f"dA{i}"], e[f"dB{i}"] = lay.be.bwd_rs(lay, seg_off, seg_task, e[src])
                lay.release_ag()
            comp(f"bwd{i}", (g,), (f"dX{i}", f"dA{i}", f"dB{i}"), bwd, flops_per_layer[i])
            comm(f"AR(dA{i})", (f"dA{i}",), (f"dA{i}:sum",), lambda e, i=i: all_reduce_async(e[f"dA{i}"], group))
            g = f"dX{i}"
        elif kind == "col":
            def bwd(e, i=i, src=g, lay=lay):
                dXp, dA, dB = lay.be.bwd(seg_off, seg_task, lay.ads, e[src], lay.X, lay.W, lay.Hs, lay.r_cap)
                e[f"dXp{i}"], e[f"dA{i}"], e[f"dB{i}"] = dXp, dA, dB
                if hasattr(lay, "release_ag"):
                    lay.release_ag()
            comp(f"bwd{i}", (g,), (f"dXp{i}", f"dA{i}", f"dB{i}"), bwd, flops_per_layer[i])
            comm(f"AR(dA{i})", (f"dA{i}",), (f"dA{i}:sum",), lambda e, i=i: all_reduce_async(e[f"dA{i}"], group))

            def rs(e, i=i):
                d = e[f"dXp{i}"]
                p = dist.get_world_size(group)
                out = torch.empty((d.shape[0] // p,) + tuple(d.shape[1:]), dtype=d.dtype, device=d.device)
                e[f"dX{i}"] = out
                return reduce_scatter_rows_async(d, out, group)
            comm(f"RS(dx{i})", (f"dXp{i}",), (f"dX{i}",), rs)
            g = f"dX{i}"
        elif getattr(lay, "fused_ag", False):
            def bwd(e, i=i, src=g, lay=lay):
                e[f"dX{i}"], e[f"dA{i}"], e[f"dB{i}"] = lay.be.bwd_ag(lay, seg_off, seg_task, e[src])
            comp(f"bwd{i}", (g,), (f"dX{i}", f"dA{i}", f"dB{i}"), bwd, flops_per_layer[i])
            comm(f"AR(dB{i})", (f"dB{i}",), (f"dB{i}:sum",), lambda e, i=i: all_reduce_async(e[f"dB{i}"], group))
            g = f"dX{i}"
        else:
            def ag(e, i=i, src=g):
                d = e[src]
                p = dist.get_world_size(group)
                out = torch.empty((d.shape[0] * p,) + tuple(d.shape[1:]), dtype=d.dtype, device=d.device)
                e[f"dYg{i}"] = out
                return all_gather_rows_async(d, out, group)
            comm(f"AG(dy{i})", (g,), (f"dYg{i}",), ag)

            def bwd(e, i=i, lay=lay):
                dXp, dA, dB = lay.be.bwd(seg_off, seg_task, lay.ads, e[f"dYg{i}"], lay.X, lay.W, lay.Hs,
                                         lay.r_cap)
                e[f"dX{i}"], e[f"dA{i}"], e[f"dB{i}"] = dXp, dA, dB
            comp(f"bwd{i}", (f"dYg{i}",), (f"dX{i}", f"dA{i}", f"dB{i}"), bwd, flops_per_layer[i])
            comm(f"AR(dB{i})", (f"dB{i}",), (f"dB{i}:sum",), lambda e, i=i: all_reduce_async(e[f"dB{i}"], group))
            g = f"dX{i}"
    return ops
