"""CPU oracle (test infrastructure only -- never imported by the product path).

See `oracle/dualkv_oracle.py` for the restated reference algorithm and its
file:line citations.  Pinned against the reference's own outputs by
`tests/test_oracle_golden.py` (fixtures from `tools/make_golden.py`).
"""
from .dualkv_oracle import *  # noqa: F401,F403
