"""paper_2505_24034_b200 -- `llrl`: B200-native DDMA trainer->generator weight
synchronisation (LlamaRL, arxiv 2505.24034 §5.2).

The product is ``libllrl.so`` (C ABI, include/llrl.h), built in-tree by
``build.py``; ``llrl`` is its ctypes binding (importing it raises if the
library is missing -- there is no fallback) and ``runner`` the torch plumbing
(device buffers, streams, process groups, IPC exchange) used by the tests and
bench.py.
"""
