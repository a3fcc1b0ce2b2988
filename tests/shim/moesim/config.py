import sys

import paper_2510_10302_b200.config as _impl

sys.modules[__name__] = _impl
