"""B200-native merged multi-model inference (GEMEL, arXiv 2201.07705).

  gemel    -- ctypes binding of the C ABI (include/gemel.h)
  engine   -- MergedWorkload: arenas, streams and the per-step call (torch for memory only)
  build    -- nvcc build of libgemel.so for sm_100a
"""
