"""Exception types with the reference's names and ValueError bases, so callers'
`except` clauses keep working (sf/tensor_core.py:15, sf/block_sparse.py:18,
sf/neuron_ops.py:18, sf/patterns.py:20, sf/autograd.py:24, sf/harness.py:28)."""


class ShapeError(ValueError):
    """Operand shapes are incompatible (sf/tensor_core.py:15)."""


class LayoutError(ValueError):
    """Layout inconsistent with operand shapes or softmax preconditions (sf/block_sparse.py:18)."""


class MaskError(ValueError):
    """Neuron-block mask inconsistent with weight shapes (sf/neuron_ops.py:18)."""


class PatternError(ValueError):
    """Invalid pattern parameter or unknown pattern id (sf/patterns.py:20)."""


class GradientError(ValueError):
    """Gradient set inconsistent with the trainable parameter set (sf/autograd.py:24)."""


class ConfigError(ValueError):
    """Malformed run configuration (sf/harness.py:28)."""


class UnsupportedError(ValueError):
    """Shape outside the envelope of the sm_100a kernels (no CPU fallback exists)."""


class CudaError(RuntimeError):
    """A CUDA launch or driver call inside the extension failed."""
