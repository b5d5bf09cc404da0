"""Fused PARALLEL streaming-tile template instantiation (placeholder)."""


def emit(kname, plan, kplan, ctype, dtypes):
    raise NotImplementedError("pfused kernels are not implemented yet")
