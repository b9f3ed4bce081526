"""paper_2506_12761_b200 -- B200-native batched TFHE gate bootstrapping for VeLoPIR (arXiv 2506.12761).

The product is libvlp.so (include/vlp.h): sm_100a CUDA kernels for blind rotation / sample extraction /
key switching, a C++ level scheduler for the IntV / CoV / IdM circuits, and the host client calls.  This
package is its Python binding (argument marshalling only); there is no CPU fallback.
"""
from . import _lib  # noqa: F401
from .api import Keys, Program, Server, meta, record_cts, to_device, to_host  # noqa: F401
