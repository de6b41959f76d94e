"""Domain types, mirroring the reference's dataclasses field for field.

GrayFrame / PyramidLayer / ScaleSpacePyramid   pyramid.py:20-64
Candidate / Keypoint                           detector.py:36-55
DetectionMask / SubsampledMask / Feature       masking.py:30-63
MaskConfig                                     masking.py:66-81
PipelineConfig / FrameReport                   pipeline.py:46-71
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

OCTAVE = "octave"
INTRA = "intra"
DETECTED = "detected"
PROPAGATED = "propagated"

DEFAULT_THRESHOLD = 55  # detector.py:32
RETRIEVAL_THRESHOLD = 70  # detector.py:33
DEFAULT_INTENSITY_THRESHOLD = 20.0  # masking.py:26
DEFAULT_BINNING_GRID = (16, 16)  # masking.py:27


@dataclass(frozen=True, eq=False)
class GrayFrame:
    """A single 8-bit grayscale frame (row-major) plus its frame number."""

    data: np.ndarray
    index: int = 0

    def __post_init__(self):  # pyramid.py:27-33
        if not isinstance(self.data, np.ndarray) or self.data.ndim != 2:
            raise ValueError("frame data must be a 2-D array")
        if self.data.dtype != np.uint8:
            raise ValueError("frame data must be uint8")
        if self.data.shape[0] < 1 or self.data.shape[1] < 1:
            raise ValueError("frame dimensions must be positive")

    @property
    def height(self) -> int:
        return self.data.shape[0]

    @property
    def width(self) -> int:
        return self.data.shape[1]


@dataclass(frozen=True, eq=False)
class PyramidLayer:
    frame: GrayFrame
    scale: float
    kind: str
    level: int


@dataclass(eq=False)
class ScaleSpacePyramid:
    """Layers ordered by strictly decreasing scale: o0, i0, o1, i1, ..."""

    layers: list[PyramidLayer]
    n_octaves: int

    def layer_at(self, kind: str, level: int) -> GrayFrame:
        for layer in self.layers:
            if layer.kind == kind and layer.level == level:
                return layer.frame
        raise KeyError(f"no {kind} layer at level {level}")


@dataclass(frozen=True, slots=True)
class Candidate:
    x: int
    y: int
    layer_id: tuple[str, int]
    score: int


@dataclass(frozen=True, slots=True)
class Keypoint:
    """Sub-pixel keypoint in original-frame coordinates (theta 0 until described)."""

    x: float
    y: float
    sigma: float
    theta: float = 0.0
    score: float = 0.0


@dataclass(frozen=True, eq=False)
class DetectionMask:
    """Full-frame binary grid; detection runs only where bits are 1."""

    bits: np.ndarray

    @property
    def width(self) -> int:
        return self.bits.shape[1]

    @property
    def height(self) -> int:
        return self.bits.shape[0]

    @property
    def coverage(self) -> float:
        return float(self.bits.mean())


@dataclass(frozen=True, eq=False)
class SubsampledMask:
    """Cell-resolution mask; cell size in pixels is bound when known."""

    bits: np.ndarray
    cell_w: int | None = None
    cell_h: int | None = None


@dataclass(frozen=True, eq=False, slots=True)
class Feature:
    kp: Keypoint
    desc: np.ndarray  # 512-element 0/1 uint8 vector
    origin: str = DETECTED
    age: int = 0


@dataclass(frozen=True)
class MaskConfig:
    mode: str = "none"  # none | intensity | binning | temporal
    t_i: float = DEFAULT_INTENSITY_THRESHOLD
    t_h: int = 1
    grid: tuple[int, int] = DEFAULT_BINNING_GRID
    octave_for_mask: int | None = None
    per_layer: bool = False

    def __post_init__(self):  # masking.py:75-81
        if self.mode not in ("none", "intensity", "binning", "temporal"):
            raise ValueError(f"unknown mask mode {self.mode!r}")
        if self.t_h < 0:
            raise ValueError("histogram threshold must be >= 0")
        if self.grid[0] < 1 or self.grid[1] < 1:
            raise ValueError("binning grid must be at least 1x1")


@dataclass(frozen=True)
class GopConfig:
    """temporal.py:23-43: the block-matching baseline's GOP and search parameters."""

    delta: int = 10  # GOP length
    patch: int = 16  # patch side length, pixels
    t_bm: float = 1800.0  # SAD accept threshold
    t_et: float = 1000.0  # early-termination SAD threshold
    coarse_window: float = 12.0  # search extends +/- this many pixels
    coarse_step: float = 2.0
    fine_window: float = 1.75  # refinement extends +/- this around the coarse winner
    fine_step: float = 0.25

    def __post_init__(self):
        if self.delta < 1:
            raise ValueError("GOP length must be >= 1")
        if self.patch % 2 != 0 or self.patch < 2:
            raise ValueError("patch side must be even and positive")
        if self.fine_step > self.coarse_step:
            raise ValueError("fine_step must not exceed coarse_step")
        if self.t_bm <= 0 or self.t_et <= 0:
            raise ValueError("SAD thresholds must be positive")


@dataclass(frozen=True)
class PipelineConfig:
    threshold: int = DEFAULT_THRESHOLD
    n_octaves: int = 4
    mask: MaskConfig = field(default_factory=MaskConfig)
    gop: GopConfig = field(default_factory=GopConfig)  # temporal mode (pipeline.py:52)
    match: object = None  # MatchConfig (matching is downstream of this path)
    seed: int = 0
    parallel: bool = False  # accepted and ignored: the device path is always parallel


@dataclass
class FrameReport:
    frame: int
    n_detected: int
    n_propagated: int
    n_total: int
    coverage: float
    t_pyramid_ms: float
    t_mask_ms: float
    t_detect_ms: float
    t_describe_ms: float
    t_total_ms: float
    t_wall_ms: float = 0.0
    n_dropped: int = 0
    accuracy: float | None = None
