"""paper_2510_19689_b200 — B200-native TabNet batch predict + feature-mask explain.

Drop-in for the reference's ``tabserve.model`` inference API
(``tabserve/model/__init__.py:1-12``): same names, argument meaning and error
types, with ``TabNetModel.apply`` running as one fused sm_100a kernel.
Training (``train``, ``TrainingSchedule``) is out of scope; its
evaluation helpers ``accuracy``/``roc_auc`` (training.py:177-202) are callers of
``apply`` and live in ``metrics``.
"""
from .config import ModelConfig
from .errors import (ChecksumError, ConfigurationError, DeviceError, FormatVersionError,
                     InvalidInputError, ModelFormatError, TabserveError, TrainingError,
                     TruncatedStreamError, UnsupportedShapeError)
from .metrics import accuracy, roc_auc
from .network import (DEFAULT_PRECISION, Explanation, ForwardResult, GpuTabNetModel,
                      PredictionOutput, TabNetModel, TabNetRegressor, init_parameters)
from .sparsemax import project_simplex_bruteforce, sparsemax
from .io import load_model, load_model_file, save_model, save_model_file

__version__ = "0.1.0"

__all__ = [
    "ModelConfig", "TabNetModel", "GpuTabNetModel", "TabNetRegressor", "Explanation", "PredictionOutput",
    "ForwardResult", "init_parameters", "sparsemax", "project_simplex_bruteforce",
    "save_model", "load_model", "save_model_file", "load_model_file", "DEFAULT_PRECISION",
    "accuracy", "roc_auc",
    "TabserveError", "InvalidInputError", "ConfigurationError", "ModelFormatError",
    "FormatVersionError", "TruncatedStreamError", "ChecksumError", "DeviceError",
    "UnsupportedShapeError", "TrainingError",
]
