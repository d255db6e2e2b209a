"""ORACLE -- test infrastructure only (see oracle/hht_oracle.c header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs may
import this package. The product path (paper_1007_0547_b200) never imports it.
"""
from .oracle import (ALPHA, BETA, OracleResult, build, circle_mb_passes, circle_passes, code,  # noqa: F401
                     corner_below, dense_votes, detect, detect_removal, detect_subtree, generic_code, region_votes)
from .frontend import edges, partition_edges, sobel  # noqa: F401
