"""B200-native mini-batch gradient oracle (the hot path of BurTorch, arXiv 2503.13795).

A recorded scalar tape (reference tapegrad API) is compiled once and evaluated
for a whole batch on the GPU: forward sweep, reverse sweep, batch reduction
and GD update.  See DESIGN.md.
"""
from ._lib import DomainError, InvalidArgument, TgError  # noqa: F401  (raises if libtg.so is missing)
from .tape import (  # noqa: F401
    MODELS, OpKind, Pipeline, Program, Tape, TapeDesc, build_model, op_name, synth_batch, synth_ctr, synth_ctr_device,
)
