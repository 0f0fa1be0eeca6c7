"""B200-native (sm_100a) implementation of the permez block-parallel PW_REL
compress/decompress path (arXiv 2309.09778).

Public entry points mirror the reference package: ``compress`` /
``decompress`` (pipeline), the transform module, the exception hierarchy.
"""
from . import errors, transform
from .errors import PermezError
from .pipeline import (Codec, CompressConfig, CompressInfo, GraphedCompressor, PipelinedCompressor,
                       PipelinedDecompressor, compress, decompress)
from .hostpipe import HostPipeline
from .predictor import PerceptronModel, init_model, lorenzo_coefficients

__all__ = ["compress", "decompress", "Codec", "HostPipeline", "GraphedCompressor", "PipelinedCompressor", "PipelinedDecompressor", "CompressConfig", "CompressInfo", "PerceptronModel", "init_model",
           "lorenzo_coefficients", "errors", "transform", "PermezError"]
