"""B200-native hot path of Least-Loaded Expert Parallelism (LLEP, arxiv 2601.17111).

The product is the C-ABI library `libllep.so` (include/llep.h, sources in csrc/); `llep` is its
thin ctypes binding.  Build with `python -m paper_2601_17111_b200.build`.
"""
