"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the compression method (no LM, no softmax,
no N-gram, no quantizer, no coder).  It only produces:

* a synthetic token vocabulary (``vocab.py``),
* alice29-/enwik8-shaped synthetic text (``text.py``; SURVEY.md §8(d) recipe),
* a random-init SmolLM2-135M-shaped weight file in our flat ``NCW1`` format
  (``weights.py``),

all deterministic functions of a seed.  Both the CPU oracle (``oracle/``) and
the CUDA product path read the same bytes; neither generates them.
"""
from .configs import ModelShape, SHAPES, WORKLOADS, Workload  # noqa: F401
from .vocab import make_vocab  # noqa: F401
from .text import make_text  # noqa: F401
from .weights import write_ncw, ensure_model, ensure_text, cache_dir  # noqa: F401
