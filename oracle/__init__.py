"""ORACLE — test infrastructure only (see oracle/hc_oracle.c header).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import this package.  The product package
``paper_2310_15711_b200`` never imports it, and it never imports the product.
"""
from .oracle import (  # noqa: F401
    build, lib_path, shift, hash_qgram, link_hash, preprocess, hc_search,
    hc_search_segmented, shc_search, brute, brute_threaded, hc_threaded,
    Metrics,
)
