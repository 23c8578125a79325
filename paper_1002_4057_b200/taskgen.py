"""Task streams of the three-step tile inversion -- same API as the reference
`tileinv.taskgen` (taskgen.py:31-282).

Streams are generated natively (csrc/api.cu `tinv_gen_stream`, the loop
nests of taskgen.py:178-223) into a compact int32 task table that the device
executor consumes directly; the reference-shaped `Task` objects are
materialized lazily, only when `stream.tasks` is read.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from . import _native
from .kernels import KernelKind
from .tile_matrix import InvalidSizeError, TileId


class Mode(enum.Enum):
    READ = "R"
    READWRITE = "RW"
    WRITE = "W"  # working-array copies only


class Step(enum.Enum):
    CHOLESKY = "1"
    TRINV = "2"
    PRODUCT = "3"
    COPY = "copy"


class Placement(enum.Enum):
    IN_PLACE = "in"
    OUT_OF_PLACE = "out"


@dataclass(frozen=True)
class Access:
    tile: TileId
    mode: Mode


@dataclass(frozen=True)
class Task:
    """One tile-kernel invocation; reads in operand order, output last
    (taskgen.py:55-87). kind is None for copy tasks."""

    id: int
    kind: KernelKind | None
    indices: tuple
    accesses: tuple
    step: Step

    @property
    def is_copy(self) -> bool:
        return self.step is Step.COPY

    @property
    def output(self) -> Access:
        return self.accesses[-1]

    @property
    def reads(self) -> tuple:
        return self.accesses[:-1]

    @property
    def kind_name(self) -> str:
        return "COPY" if self.kind is None else self.kind.value

    def __str__(self) -> str:
        return f"{self.kind_name}({','.join(str(i) for i in self.indices)})"


def parse_loops(loops: str) -> str:
    """taskgen.py:90-94."""
    if len(loops) != 3 or any(ch not in "UD" for ch in loops):
        raise ValueError(f"loop order must match [UD]{{3}}, got {loops!r}")
    return loops


DEFAULT_LOOPS = "UDU"


@dataclass(frozen=True)
class VariantConfig:
    """taskgen.py:105-121."""

    placement: Placement = Placement.IN_PLACE
    loops: str = DEFAULT_LOOPS
    pipelined: bool = True
    workers: int = 1

    def __post_init__(self):
        parse_loops(self.loops)
        if self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")

    def describe(self) -> str:
        pipe = "pipelined" if self.pipelined else "barriered"
        return f"{self.placement.value}-place {self.loops} {pipe}"


# ---- table <-> Task codes (include/tileinv_b200.h)
KIND_CODE = {None: 0, KernelKind.POTRF: 1, KernelKind.TRSM: 2, KernelKind.SYRK_SUB: 3, KernelKind.SYRK_ADD_T: 4,
             KernelKind.GEMM: 5, KernelKind.TRTRI: 6, KernelKind.TRMM_LEFT: 7, KernelKind.TRMM_RIGHT_NEG: 8,
             KernelKind.TRMM_LEFT_T: 9, KernelKind.LAUUM: 10}
CODE_KIND = {v: k for k, v in KIND_CODE.items()}
STEP_CODE = {Step.COPY: 0, Step.CHOLESKY: 1, Step.TRINV: 2, Step.PRODUCT: 3}
CODE_STEP = {v: k for k, v in STEP_CODE.items()}
NIDX = {0: 2, 1: 1, 2: 2, 3: 2, 4: 2, 5: 3, 6: 1, 7: 2, 8: 2, 9: 2, 10: 1}
NATIVE_LABELS = ("A", "B", "C")


class TaskStream:
    """Ordered task list plus barrier positions (taskgen.py:124-146).

    Natively generated streams keep their int32 task table (`_table`) and
    build `tasks` on first access; user-built streams are encoded on demand."""

    def __init__(self, tasks=None, barriers=None, t: int = 0, steps: tuple = (),
                 placement: Placement = Placement.IN_PLACE, loops: str = DEFAULT_LOOPS):
        self._tasks = list(tasks) if tasks is not None else []
        self.barriers = set(barriers) if barriers else set()
        self.t = t
        self.steps = steps
        self.placement = placement
        self.loops = loops
        self._table = None
        self._labels = None

    @classmethod
    def _native(cls, table, barriers, t, steps, placement, loops):
        s = cls(None, set(int(b) for b in barriers), t, steps, placement, loops)
        s._tasks = None
        s._table = table
        s._labels = NATIVE_LABELS
        return s

    @property
    def tasks(self):
        if self._tasks is None:
            self._tasks = decode_tasks(self._table, self._labels)
        return self._tasks

    @tasks.setter
    def tasks(self, value):
        self._tasks = list(value)
        self._table = None

    def __len__(self):
        return len(self._table) if self._tasks is None else len(self._tasks)

    @property
    def pipelined(self) -> bool:
        return not self.barriers

    def describe(self) -> str:
        names = "+".join(s.value for s in self.steps)
        pipe = "pipelined" if self.pipelined else "barriered"
        return f"step {names} {self.placement.value}-place {self.loops} {pipe} t={self.t}"

    def __eq__(self, other):
        if not isinstance(other, TaskStream):
            return NotImplemented
        return (self.tasks == other.tasks and self.barriers == other.barriers and self.t == other.t
                and self.steps == other.steps and self.placement == other.placement and self.loops == other.loops)

    def __repr__(self):
        return f"TaskStream({len(self)} tasks, {self.describe()})"

    def table(self, matrix_label: str = "A"):
        """int32 task table (n, 16) with the matrix label mapped to 0 and the
        other labels to 1, 2, ... (first appearance)."""
        if self._table is not None and self._labels and self._labels[0] == matrix_label:
            return self._table
        return encode_tasks(self.tasks, matrix_label)


def decode_tasks(table, labels):
    out = []
    for tid, f in enumerate(table.tolist()):
        kind = CODE_KIND[f[0]]
        step = CODE_STEP[f[1]]
        idx = tuple(f[2:2 + NIDX[f[0]]])
        acc = []
        if f[9] >= 1:
            acc.append(Access(TileId(labels[f[10]], f[11], f[12]), Mode.READ))
        if f[9] >= 2:
            acc.append(Access(TileId(labels[f[13]], f[14], f[15]), Mode.READ))
        acc.append(Access(TileId(labels[f[5]], f[6], f[7]), Mode.WRITE if f[8] == 2 else Mode.READWRITE))
        out.append(Task(tid, kind, idx, tuple(acc), step))
    return out


def encode_tasks(tasks, matrix_label="A"):
    labels = {matrix_label: 0}
    rows = np.full((len(tasks), _native.TASK_FIELDS), -1, dtype=np.int32)
    for n, task in enumerate(tasks):
        r = rows[n]
        r[0] = KIND_CODE.get(task.kind, -1)
        r[1] = STEP_CODE[task.step]
        for x, v in enumerate(task.indices[:3]):
            r[2 + x] = v
        out = task.output
        r[5] = labels.setdefault(out.tile.label, len(labels))
        r[6], r[7] = out.tile.row, out.tile.col
        r[8] = 2 if out.mode is Mode.WRITE else 1
        reads = task.reads
        r[9] = len(reads)
        for x, a in enumerate(reads[:2]):
            r[10 + 3 * x] = labels.setdefault(a.tile.label, len(labels))
            r[11 + 3 * x], r[12 + 3 * x] = a.tile.row, a.tile.col
    return rows


def _check_t(t: int):
    if t < 1:
        raise InvalidSizeError(f"tile count must be >= 1, got {t}")


def _gen(t, mask, loops, placement, pipelined, steps):
    _check_t(t)
    table, bars = _native.gen_stream(t, mask, loops, placement is Placement.OUT_OF_PLACE, pipelined)
    return TaskStream._native(table, bars, t, steps, placement, loops if len(loops) == 3 else loops * 3)


def gen_step1(t: int, direction: str = "U") -> TaskStream:
    """Tile Cholesky factorization (taskgen.py:230-235)."""
    parse_loops(direction * 3)
    return _gen(t, 1, direction * 3, Placement.IN_PLACE, True, (Step.CHOLESKY,))


def gen_step2(t: int, direction: str = "D", placement: Placement = Placement.IN_PLACE) -> TaskStream:
    """Tile inversion of the lower factor (taskgen.py:238-244)."""
    parse_loops(direction * 3)
    return _gen(t, 2, direction * 3, placement, True, (Step.TRINV,))


def gen_step3(t: int, direction: str = "U", placement: Placement = Placement.IN_PLACE) -> TaskStream:
    """Product of the inverted factor with its transpose (taskgen.py:247-253)."""
    parse_loops(direction * 3)
    return _gen(t, 4, direction * 3, placement, True, (Step.PRODUCT,))


def gen_inversion(t: int, config: VariantConfig) -> TaskStream:
    """Full three-step stream; barriers between steps unless pipelined (taskgen.py:256-269)."""
    return _gen(t, 7, config.loops, config.placement, config.pipelined,
                (Step.CHOLESKY, Step.TRINV, Step.PRODUCT))


def format_stream(stream: TaskStream) -> str:
    """`<id> <step> <kind>(<indices>) R:<tiles> RW:<tile>` lines (taskgen.py:272-282)."""
    lines = []
    for task in stream.tasks:
        if task.id in stream.barriers:
            lines.append("BARRIER")
        reads = ",".join(str(a.tile) for a in task.reads) or "-"
        lines.append(f"{task.id} {task.step.value} {task} R:{reads} RW:{task.output.tile}")
    return "\n".join(lines) + "\n"
