"""Host-side schedule tables and the analytic pipeline trace.

``moe_forward`` returns ``(y, PipelineTrace)`` like the reference
(``pipeline.py:572-615``).  The device path counts nothing at run time; the
trace is replayed on the host from the expert histogram, exactly as the
reference's ``trace_from_counts`` does (``pipeline.py:534-565``), which the
reference's own tests pin equal to an executed trace.  Also here: the host
versions of ``expert_offsets`` and ``build_block_schedule`` used for the
trace and for cross-checking the device tile table.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import IndexOutOfRange, InvalidBlockM, ScheduleMismatch, ShapeMismatch
from .types import BlockSchedule, ExpertOffsets, ModelConfig, PipelineParams

STAGE_ROUTER = "Router"
STAGE_HOST_SCHEDULE = "HostSchedule"
STAGE_PERMUTE = "Permute"
STAGE_GATE_UP = "GateUp"
STAGE_DOWN = "Down"
STAGE_UNPERMUTE = "Unpermute"
DEVICE_STAGES = (STAGE_ROUTER, STAGE_PERMUTE, STAGE_GATE_UP, STAGE_DOWN, STAGE_UNPERMUTE)
INDEX_BYTES = 8  # the reference charges int64 indices


@dataclass
class StageRecord:
    """Tile/FLOP/byte counters for one stage (``pipeline.py:81-106``)."""

    stage: str
    tiles: int = 0
    flops: int = 0
    reads: dict = field(default_factory=dict)
    writes: dict = field(default_factory=dict)

    @property
    def bytes_read(self) -> int:
        return sum(self.reads.values())

    @property
    def bytes_written(self) -> int:
        return sum(self.writes.values())

    @property
    def total_bytes(self) -> int:
        return self.bytes_read + self.bytes_written


@dataclass
class PipelineTrace:
    """Ordered stage records for one forward pass (``pipeline.py:109-131``)."""

    element_bytes: int
    records: list = field(default_factory=list)

    def add(self, record: StageRecord) -> None:
        self.records.append(record)

    def stage(self, name: str) -> StageRecord:
        for r in self.records:
            if r.stage == name:
                return r
        raise KeyError(f"no record for stage {name!r}")

    @property
    def total_flops(self) -> int:
        return sum(r.flops for r in self.records)

    @property
    def total_bytes(self) -> int:
        return sum(r.total_bytes for r in self.records)


def expert_offsets(counts) -> ExpertOffsets:
    """Exclusive prefix sum (``scheduler.py:85-94``)."""
    counts = np.asarray(counts, dtype=np.int64)
    if counts.ndim != 1:
        raise ShapeMismatch("histogram must be 1-D")
    if counts.size and counts.min() < 0:
        raise IndexOutOfRange("histogram counts must be non-negative")
    off = np.zeros(counts.size + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    return ExpertOffsets(offsets=off)


def build_block_schedule(offsets: ExpertOffsets, block_m: int) -> BlockSchedule:
    """Algorithm 1 tile list (``scheduler.py:106-117``)."""
    if not isinstance(block_m, (int, np.integer)) or isinstance(block_m, bool):
        raise InvalidBlockM(f"block_m must be an integer, got {block_m!r}")
    if block_m < 1:
        raise InvalidBlockM(f"block_m must be >= 1, got {block_m}")
    off = np.asarray(offsets.offsets)
    entries = []
    for e in range(off.size - 1):
        n_e = int(off[e + 1] - off[e])
        entries.extend((e, s) for s in range(0, n_e, block_m))
    return BlockSchedule(entries=tuple(entries), block_m=int(block_m))


def check_schedule(offsets: ExpertOffsets, schedule: BlockSchedule) -> None:
    """Raise ScheduleMismatch unless ``schedule`` tiles ``offsets`` (``pipeline.py:143-150``)."""
    expected = build_block_schedule(offsets, schedule.block_m)
    if sorted(schedule.entries) != sorted(expected.entries):
        raise ScheduleMismatch(
            f"schedule ({len(schedule.entries)} entries) does not tile the given offsets "
            f"(expected {len(expected.entries)} entries)"
        )


def _steps(total: int, block: int) -> int:
    return math.ceil(total / block) if total else 0


def _spans(off: np.ndarray, block_m: int):
    for e in range(off.size - 1):
        n_e = int(off[e + 1] - off[e])
        for s in range(0, n_e, block_m):
            yield min(block_m, n_e - s)


def trace_from_counts(config: ModelConfig, batch: int, counts, params: PipelineParams) -> PipelineTrace:
    """Replay the six-record accounting from a histogram (``pipeline.py:534-565``).

    Stage records follow ``pipeline.py:406-531`` (router, host schedule,
    permute, gate+up fused/unfused, down, unpermute).
    """
    counts = np.asarray(counts, dtype=np.int64)
    if counts.shape != (config.num_experts,):
        raise ShapeMismatch(f"histogram has shape {counts.shape}, expected ({config.num_experts},)")
    if int(counts.sum()) != batch * config.top_k:
        raise ShapeMismatch(
            f"histogram sums to {int(counts.sum())}, expected B*k = {batch * config.top_k}"
        )
    eb = config.element_bytes
    d, e, f, k = config.hidden_dim, config.num_experts, config.ffn_dim, config.top_k
    offsets = expert_offsets(counts)
    off = offsets.offsets
    total = int(off[-1])
    schedule = build_block_schedule(offsets, params.block_m)
    spans = list(_spans(off, params.block_m))
    tr = PipelineTrace(element_bytes=eb)
    tr.add(StageRecord(
        stage=STAGE_ROUTER, tiles=0, flops=2 * batch * d * e + 4 * batch * e,
        reads={"input": batch * d * eb, "weight": d * e * eb},
        writes={"scores": batch * e * eb, "route_weights": batch * k * eb, "index": batch * k * INDEX_BYTES}))
    tr.add(StageRecord(stage=STAGE_HOST_SCHEDULE, tiles=len(schedule.entries)))
    tr.add(StageRecord(
        stage=STAGE_PERMUTE, tiles=0, flops=0,
        reads={"input": total * d * eb, "index": total * INDEX_BYTES},
        writes={"output": total * d * eb}))
    # gate + up
    ks, ns = _steps(d, params.block_k), _steps(f, params.block_n)
    streams = 1 if params.fused else 2
    tiles = sum(streams * ks * ns for _ in spans)
    inp = sum(streams * m * d for m in spans)
    wts = sum(2 * d * f for _ in spans)
    wr = sum(m * f for m in spans)
    gflops = sum(4 * m * d * f for m in spans)
    if params.fused:
        tr.add(StageRecord(stage=STAGE_GATE_UP, tiles=tiles, flops=gflops + 5 * wr,
                           reads={"input": inp * eb, "weight": wts * eb},
                           writes={"intermediate": wr * eb}))
    else:
        tr.add(StageRecord(stage=STAGE_GATE_UP, tiles=tiles, flops=gflops + 5 * total * f,
                           reads={"input": inp * eb, "weight": wts * eb, "buffer": 2 * total * f * eb},
                           writes={"gate_out": wr * eb, "up_out": wr * eb, "intermediate": total * f * eb}))
    # down
    ks, ns = _steps(f, params.block_k), _steps(d, params.block_n)
    tr.add(StageRecord(
        stage=STAGE_DOWN, tiles=sum(ks * ns for _ in spans), flops=sum(2 * m * f * d for m in spans),
        reads={"input": sum(m * f for m in spans) * eb, "weight": sum(f * d for _ in spans) * eb},
        writes={"output": sum(m * d for m in spans) * eb}))
    tr.add(StageRecord(
        stage=STAGE_UNPERMUTE, tiles=0, flops=2 * batch * k * d,
        reads={"input": batch * k * d * eb, "index": batch * k * INDEX_BYTES, "route_weights": batch * k * eb},
        writes={"output": batch * d * eb}))
    return tr


# ---------------------------------------------------------------------------
# Minimal-traffic model (perfmodel.py:196-249): the algorithmic bytes/FLOPs
# that the bench's roofline fractions divide by.
# ---------------------------------------------------------------------------

def stage_flops(stage: str, config: ModelConfig, batch: int) -> int:
    d, e, f, k = config.hidden_dim, config.num_experts, config.ffn_dim, config.top_k
    t = batch * k
    return {
        STAGE_ROUTER: 2 * batch * d * e + 4 * batch * e,
        STAGE_PERMUTE: 0,
        STAGE_GATE_UP: 4 * t * d * f + 5 * t * f,
        STAGE_DOWN: 2 * t * f * d,
        STAGE_UNPERMUTE: 2 * t * d,
    }[stage]


def stage_bytes(stage: str, config: ModelConfig, batch: int, counts, element_bytes=None) -> int:
    counts = np.asarray(counts, dtype=np.int64)
    eb = config.element_bytes if element_bytes is None else element_bytes
    d, e, f, k = config.hidden_dim, config.num_experts, config.ffn_dim, config.top_k
    total = int(counts.sum())
    active = int(np.count_nonzero(counts))
    if stage == STAGE_ROUTER:
        return (batch * d + d * e + batch * e + batch * k) * eb + batch * k * INDEX_BYTES
    if stage == STAGE_PERMUTE:
        return 2 * total * d * eb + total * INDEX_BYTES
    if stage == STAGE_GATE_UP:
        return (total * d + total * f) * eb + 2 * active * d * f * eb
    if stage == STAGE_DOWN:
        return (total * f + total * d) * eb + active * f * d * eb
    if stage == STAGE_UNPERMUTE:
        return (total * d + total + batch * d) * eb + total * INDEX_BYTES
    raise ValueError(stage)


# ---------------------------------------------------------------------------
# Activation-traffic comparison of the fused and unfused gate+up
# (perfmodel.py:70-96 TrafficSource / TrafficReport, :122-180), plus the
# device-MEASURED source: DRAM bytes of the two variants' launches from ncu.
# ---------------------------------------------------------------------------

TRAFFIC_CLOSED_FORM = "closed_form"
TRAFFIC_TILE_TRACE = "tile_trace"
TRAFFIC_MEASURED = "measured"


@dataclass(frozen=True)
class TrafficReport:
    """Fused vs unfused gate+up activation traffic (``perfmodel.py:88-96``)."""

    unfused_bytes: int
    fused_bytes: int
    savings_bytes: int
    savings_ratio: float
    source: str


def _report(unfused: int, fused: int, source: str) -> TrafficReport:
    savings = unfused - fused
    return TrafficReport(unfused_bytes=int(unfused), fused_bytes=int(fused), savings_bytes=int(savings),
                         savings_ratio=savings / unfused if unfused else 0.0, source=source)


def activation_traffic_closed_form(expanded_tokens: int, ffn_dim: int, hidden_dim: int,
                                   element_bytes: int = 2) -> TrafficReport:
    """``perfmodel.py:122-145``: unfused moves ``s(4TF + 2Td)``, fused ``s(TF + Td)``."""
    t, f, d, s = int(expanded_tokens), int(ffn_dim), int(hidden_dim), int(element_bytes)
    if min(t, f, d, s) < 0 or f == 0 or d == 0 or s == 0:
        raise ValueError("dimensions must be positive (tokens may be zero)")
    return _report(s * (4 * t * f + 2 * t * d), s * (t * f + t * d), TRAFFIC_CLOSED_FORM)


def traffic_from_traces(fused_trace: "PipelineTrace", unfused_trace: "PipelineTrace") -> TrafficReport:
    """``perfmodel.py:148-180``: the same comparison from two stage traces."""
    gf = fused_trace.stage(STAGE_GATE_UP)
    gu = unfused_trace.stage(STAGE_GATE_UP)
    if "intermediate" not in gf.writes or "gate_out" in gf.writes:
        raise ShapeMismatch("first trace is not from a fused run")
    if "gate_out" not in gu.writes:
        raise ShapeMismatch("second trace is not from an unfused run")
    fused = gf.reads["input"] + gf.writes["intermediate"]
    unfused = gu.reads["input"] + gu.reads["buffer"] + gu.writes["gate_out"] + gu.writes["up_out"]
    return _report(unfused, fused, TRAFFIC_TILE_TRACE)


def traffic_from_measured(fused_dram_bytes: float, unfused_dram_bytes: float,
                          weight_bytes: float = 0.0) -> TrafficReport:
    """The comparison with MEASURED bytes: ``ncu`` dram__bytes_read + write of
    the fused gate+up launch(es) and of the unfused ones (the two projection
    launches plus the activation pass), minus the expert-weight stream both
    variants read once (``weight_bytes``, the same in both), so the report
    covers activation traffic only, as the closed form does."""
    return _report(round(unfused_dram_bytes - weight_bytes), round(fused_dram_bytes - weight_bytes),
                   TRAFFIC_MEASURED)
