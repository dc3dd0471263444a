"""B200-native (sm_100a) buffered SCPL video retargeting -- a drop-in for `vidcarve` 0.1.0.

Same public names as the reference package (pkg/src/vidcarve/__init__.py:9-68) for the
retargeting path; the compute runs in libscpl.so (include/scpl.h) with no CPU fallback.
Out of scope: media I/O, CLI, plots and the bench corpus helpers.
"""

import os as _os

# The streamed pipeline keeps up to ~13 streams busy at once (copies in/out, codes + scan,
# concurrent carve groups); with the default 8 hardware work queues, streams would share
# queues and serialise behind each other.  Takes effect if CUDA is not initialised yet.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from .batching import SeamBatch, batch_carve, default_energy, label_parents, remove_batch, select_batch
from .buffering import BufferPolicy, FixedRun, SpatioTemporalBuffer, threshold
from .energy import MAXVAL, gradient_energy, motion_energy, to_luma
from .media import MediaFormatError, read_clip_pinned, read_frames, retarget_stream, write_clip, write_frames
from .pipeline import (MODES, RetargetConfig, RunMetrics, replay_batches, retarget_image, retarget_video,
                       retarget_video_tensor, retarget_videos, scan_runs)
from .quality import SYNTHETIC_KINDS, JitterReport, SyntheticSpec, compare, format_metrics, generate, jitter
from .seams import DpTables, Seam, cumulative_energy, min_seam, remove_seam, trace_columns, transpose

__version__ = "0.1.0"

__all__ = [
    "JitterReport", "MediaFormatError", "SYNTHETIC_KINDS", "SyntheticSpec", "compare", "format_metrics", "generate",
    "jitter", "read_clip_pinned", "read_frames", "retarget_stream", "write_clip",
    "write_frames",
    "MAXVAL", "MODES", "BufferPolicy", "DpTables", "FixedRun", "RetargetConfig", "RunMetrics", "Seam",
    "SeamBatch", "SpatioTemporalBuffer", "batch_carve", "cumulative_energy", "default_energy",
    "gradient_energy", "label_parents", "min_seam", "motion_energy", "remove_batch", "remove_seam",
    "replay_batches", "retarget_image", "retarget_video", "retarget_video_tensor", "retarget_videos", "scan_runs",
    "select_batch",
    "threshold", "to_luma", "trace_columns", "transpose",
]
