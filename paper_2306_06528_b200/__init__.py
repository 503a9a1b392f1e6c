"""B200-native SVGD particle step of PusH (arXiv 2306.06528).

The product is the C-ABI library ``libpush_b200.so`` (include/push.h);
``paper_2306_06528_b200.push`` is its thin ctypes binding.
"""
from .push import (Context, PushConfig, PushError, get_unique_id, lib, local_group, make_config,  # noqa: F401
                   workspace_size)
