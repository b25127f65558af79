"""B200-native engine for the online-BP CNN hot path of arXiv 1102.0183.

Mirrors the public API of the reference package ``convkit`` for that path
(net construction, train_step / train_epoch / evaluate / run_experiment, the
``kernels`` operator seam), backed by hand-written sm_100a CUDA in
``libckb200.so`` (csrc/).  FP32 only; there is no CPU fallback.
"""

from .arch import parse_architecture, parse_experiment, resolve_geometry
from .augment import (DeformationConfig, DeformationParams, deform_channels,
                      sample_params)
from .data import (Dataset, byte_lut, from_bytes, make_glyph_dataset,
                   make_glyph_images, normalize)
from .errors import (ConfigError, ConvkitError, CudaError, DataFormatError,
                     DimensionError, GeometryError, GeometryWarning,
                     PrecisionError, StateError)
from .filters import expand_selection, filter_coefficients, make_contrast_filters
from .network import NetworkState
from .topology import (ConnectionTable, LayerSpec, NetworkSpec, build_full_table,
                       build_random_table, invert_table, output_map_size)
from .training import (EpochStats, ExperimentSummary, RunRecord, TrainConfig,
                       evaluate, init_weights, lr_at_epoch, mnist_decay,
                       predict_batch, run_experiment, run_training, targets_for,
                       train_committee_epoch, train_epoch)

__version__ = "0.1.0"
