"""Oracle: MapDevice — Eq. 7, 8, 9, Table III, Algorithm 2 (TEST INFRASTRUCTURE ONLY).

PAPER.md §III-D:
  Eq. 7  CPU_(i,j,o)   = baseCost_o * Part_(i,j) / InfPT_i
  Eq. 8  GPU_(i,j,o)   = baseCost_o * InfPT_i / Part_(i,j)
  Eq. 9  Trans_(i,j,o) = baseTransCost * Part_(i,j) / InfPT_i, baseTransCost = 0.1
  Table III base costs: Aggregation(Hash), Filtering, Shuffling 1.0;
                 Projection, Join(Hash), Expand 0.9; Scan(CSV), Sorting 0.8.
  Algorithm 2: map every operation to the GPU; traverse the DAG
  from the child (leaf) nodes; if o is the first or the last operation, or
  o-1 runs on the CPU, GPU += Trans, else CPU += Trans; if GPU > CPU map o to
  the CPU.
SPEC.md readings (R23): the DAG catalog S:153; "first" = every
leaf, "last" = the unique root, "o-1 on the CPU" = any predecessor on the CPU
(S:272-273); Part = batch bytes / NumCores; ties keep the GPU.
"""
from __future__ import annotations

SCAN, FILTER, PROJECT, HASHAGG, HASHJOIN, SORT, SHUFFLE, EXPAND = range(8)
OP_NAMES = ("Scan", "Filter", "Project", "HashAggregate", "HashJoin", "Sort", "Shuffle", "Expand")
BASE_COST = {HASHAGG: 1.0, FILTER: 1.0, SHUFFLE: 1.0, PROJECT: 0.9, HASHJOIN: 0.9, EXPAND: 0.9,
             SCAN: 0.8, SORT: 0.8}
CPU, GPU = 0, 1
INF_PT_INIT = 150e3          # 150 KB
BASE_TRANS_COST = 0.1

# DAGs: list of (op_kind, [predecessor node ids]); the last node is the root.
DAGS = {
    "LR1": [(SCAN, []), (PROJECT, [0]), (PROJECT, [0]), (HASHJOIN, [1, 2]), (PROJECT, [3])],
    "LR2": [(SCAN, []), (PROJECT, [0]), (SHUFFLE, [1]), (HASHAGG, [2]), (FILTER, [3])],
    "CM1": [(SCAN, []), (PROJECT, [0]), (SHUFFLE, [1]), (HASHAGG, [2]), (SORT, [3])],
    "CM2": [(SCAN, []), (FILTER, [0]), (SHUFFLE, [1]), (HASHAGG, [2])],
}


def dag_for(query: str):
    return DAGS[query.upper()[:3]]


def cpu_cost(base: float, part: float, infpt: float) -> float:
    if base <= 0 or part <= 0 or infpt <= 0:
        raise ValueError("non-positive cost input")
    return base * (part / infpt)


def gpu_cost(base: float, part: float, infpt: float) -> float:
    if base <= 0 or part <= 0 or infpt <= 0:
        raise ValueError("non-positive cost input")
    return base * (infpt / part)


def trans_cost(btc: float, part: float, infpt: float) -> float:
    if btc < 0 or part <= 0 or infpt <= 0:
        raise ValueError("non-positive cost input")
    return btc * (part / infpt)


def traverse(dag) -> list[int]:
    """Children-first order: DFS post-order from the root, predecessors left to right."""
    n = len(dag)
    succ_count = [0] * n
    for _, preds in dag:
        for p in preds:
            if not (0 <= p < n):
                raise ValueError("bad predecessor")
            succ_count[p] += 1
    roots = [i for i in range(n) if succ_count[i] == 0]
    if len(roots) != 1:
        raise ValueError("DAG must have exactly one root")
    order, state = [], [0] * n   # 0 new, 1 on stack, 2 done

    def visit(o):
        if state[o] == 1:
            raise ValueError("cycle")
        if state[o] == 2:
            return
        state[o] = 1
        for p in dag[o][1]:
            visit(p)
        state[o] = 2
        order.append(o)

    visit(roots[0])
    if len(order) != n:
        raise ValueError("unreachable node")
    return order


def map_device(dag, part: float, infpt: float = INF_PT_INIT, btc: float = BASE_TRANS_COST) -> list[int]:
    """Algorithm 2: per-node device (CPU=0 / GPU=1)."""
    order = traverse(dag)
    root = order[-1]
    dev = [GPU] * len(dag)
    for o in order:
        kind, preds = dag[o]
        c = cpu_cost(BASE_COST[kind], part, infpt)
        g = gpu_cost(BASE_COST[kind], part, infpt)
        t = trans_cost(btc, part, infpt)
        first = len(preds) == 0
        last = o == root
        if first or last or any(dev[p] == CPU for p in preds):
            g += t
        else:
            c += t
        if g > c:
            dev[o] = CPU
    return dev
