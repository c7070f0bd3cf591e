"""CPU oracle for the S^5 hot path -- TEST INFRASTRUCTURE ONLY.

The C restatement in ``s5_oracle.c`` follows the reference package
``strsort`` routine by routine (each function cites reference file:line).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / CPU baseline; the product path in
``paper_1305_1157_b200`` never imports it.

Pinning: ``tests/test_oracle_golden.py`` checks these functions against
fixtures produced by the reference itself (``tests/golden/make_golden.py``)
and against the reference's output digests quoted in SURVEY.md 8(d).
"""

from .oracle import *  # noqa: F401,F403
from .oracle import __all__  # noqa: F401
