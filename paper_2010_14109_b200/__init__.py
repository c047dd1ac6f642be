"""B200-native out-of-core training step of arXiv 2010.14109.

    liboocore.so   C ABI (include/oocore.h): planner, VA allocator, executor,
                   sm_100a kernels — built by `python -m paper_2010_14109_b200.build`
    binding        ctypes marshalling of that ABI
    graphs         network spec -> training-step function graph
    runtime        OutOfCoreStep: plan + pool + executor on torch CUDA streams
"""
