"""B200-native ES-RNN training / forecasting engine (drop-in for the reference's
esrnn::Trainer hot path).  Device code: csrc/ -> libesrnn_b200.so (sm_100a)."""
from .errors import *  # noqa: F401,F403
from .trainer import (BatchGradients, BenchmarkReport, Category, DatasetSplit, ForecastResult,  # noqa: F401
                      Frequency, FrequencyProfile, PerSeriesParams, SeriesRecord, TrainConfig, Trainer,
                      ValidationResult, WindowBatch, early_stop_check, make_batches, pinball_loss,
                      split_train_val_test)
from .rng import Rng  # noqa: F401

__version__ = "0.1.0"
