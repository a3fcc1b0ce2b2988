import sys

import paper_2510_10302_b200.cutoff as _impl

sys.modules[__name__] = _impl
