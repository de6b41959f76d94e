"""vidfeat-b200: B200-native (sm_100a) per-frame detect+describe hot path of
arXiv 1503.06959 ("Fast keypoint detection in video sequences"), a drop-in for
the reference package `vidfeat` 0.1.0's run_pipeline / detect / describe /
mask API.  All compute runs in hand-written CUDA kernels behind a C ABI
(include/vidfeat_b200.h); PyTorch only carries buffers and streams.

Imports are lazy so that the package (and its C-ABI symbol check) loads on a
machine without a GPU; any compute call without a CUDA device raises.
"""

from .pattern import SamplingPattern, build_default_pattern, default_pattern
from .types import (DETECTED, INTRA, OCTAVE, PROPAGATED, Candidate, DetectionMask, Feature, FrameReport, GopConfig,
                    GrayFrame,
                    Keypoint, MaskConfig, PipelineConfig, PyramidLayer, ScaleSpacePyramid, SubsampledMask)

__version__ = "0.1.0"

_LAZY = {
    "build_pyramid": "pyramid",
    "detect_candidates": "detector", "nms_and_refine": "detector", "ast_corner_score": "detector",
    "describe": "descriptor", "estimate_orientation": "descriptor", "hamming": "descriptor",
    "orientations_batch": "descriptor", "describe_batch": "descriptor",
    "intensity_diff_mask": "masking", "keypoint_binning_mask": "masking", "upsample_mask": "masking",
    "merge_features": "masking", "binning_histogram": "masking",
    "run_pipeline": "pipeline", "run_streams": "pipeline", "divergence_report": "pipeline",
    "DivergenceStat": "pipeline",
    "FeatureEngine": "engine",
    "hamming_matrix": "matching", "radius_match": "matching", "Match": "matching",
    "DEFAULT_MATCH_RADIUS": "matching", "MatchConfig": "matching", "project_points": "matching",
    "ransac_homography": "matching", "match_and_verify": "matching", "count_mpr": "matching",
    "RankedList": "evaluation", "ObjectModel": "evaluation", "ObjectEstimate": "evaluation",
    "GroundTruthRecord": "evaluation", "average_precision": "evaluation", "sequence_ap": "evaluation",
    "mean_average_precision": "evaluation", "corner_geometry": "evaluation", "locate_object": "evaluation",
    "tracking_accuracy": "evaluation", "save_ground_truth": "evaluation", "load_ground_truth": "evaluation",
    "load_relevance": "evaluation", "TRACKING_TOLERANCE_PX": "evaluation",
    "spiral_offsets": "temporal", "spiral_search": "temporal", "baseline_step": "temporal", "sad_block": "temporal",
    "dump_features": "report", "parse_features": "report", "emit_report": "report", "summarize": "report",
    "load_sequence": "io", "write_frame": "io",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    return getattr(importlib.import_module(f".{mod}", __name__), name)


__all__ = sorted(list(_LAZY) + [
    "SamplingPattern", "build_default_pattern", "default_pattern", "Candidate", "DetectionMask", "Feature", "GopConfig",
    "FrameReport", "GrayFrame", "Keypoint", "MaskConfig", "PipelineConfig", "PyramidLayer", "ScaleSpacePyramid",
    "SubsampledMask", "OCTAVE", "INTRA", "DETECTED", "PROPAGATED",
])
