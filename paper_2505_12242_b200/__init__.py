"""ZenFlow (arXiv 2505.12242) data-parallel hot path, B200-native (sm_100a).

Importance-based gradient partitioning for every linear layer's gradient:
column norms -> (NCCL) norm all-reduce -> top-k columns (cached for N steps) ->
in-place selective AdamW on the selected columns + compaction of the others ->
async D2H staging + double-buffered host accumulation.

The compute path is libzf.so (CUDA kernels, C-ABI in include/zf.h); the Python
side (``zf``) only marshals arguments.  ``zf`` is imported lazily so that
building does not require the library to exist yet.
"""

__all__ = ["zf"]


def __getattr__(name):
    if name == "zf":
        import importlib
        return importlib.import_module(__name__ + ".zf")
    raise AttributeError(name)
