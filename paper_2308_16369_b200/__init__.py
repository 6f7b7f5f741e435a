"""B200-native (sm_100a) SARATHI hybrid-batch forward pass (arXiv 2308.16369).

The product is libsarathi.so (CUDA kernels + C ABI, include/sarathi.h); ``sarathi`` is its thin
ctypes binding.  Importing ``paper_2308_16369_b200.sarathi`` fails loudly if the library is not
built — there is no CPU fallback.
"""
