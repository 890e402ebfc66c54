"""qmpm: the quantized MLS-MPM hot path of arXiv 2207.04658 on B200 (sm_100a).

The compute path is libqmpm.so (csrc/, C ABI in include/qmpm.h); `qmpm` is its
ctypes binding.  `scenes` and `schemes` hold the seeded inputs and stand-in
quantization schemes.  Importing this package loads nothing; the binding loads
the library on first use and raises if it is missing (no CPU fallback).
"""
__all__ = ["qmpm", "scenes", "schemes", "build"]
