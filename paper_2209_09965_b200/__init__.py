"""B200-native FoVolNet per-frame hot path (arXiv 2209.09965).

foveated mask + compaction -> sparse ray march -> recurrent W-Net reconstruction,
as hand-written sm_100a CUDA kernels in libfovnet.so behind a C ABI
(include/fovnet.h), with Python modules that mirror the reference package's
`fovray.sample_maps`, `fovray.renderer`, `fovray.volume`, `fovray.network`
and `fovray.bench` entry points.
"""

__version__ = "0.1.0"
