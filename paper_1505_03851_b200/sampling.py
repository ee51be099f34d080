"""Error types shared with the reference's sampling module (sampling.py:18-24)."""


class EmptyWeightsError(ValueError):
    """The weight vector is empty."""


class AllZeroError(ValueError):
    """Every weight is zero, so no outcome can be drawn."""
