"""B200-native GPipe pipeline-parallel training (arXiv 2004.09910, torchgpipe) -- Python binding of
the C-ABI library libtgp.so (include/tgp.h).  See DESIGN.md."""
from .tgp import (Pipeline, TgpError, balance, balance_by_size, balance_by_time, bench_transport,  # noqa: F401
                  exported_symbols, lib, profile_size, schedule, split)
