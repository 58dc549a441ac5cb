"""bench.py workloads (one module per BASELINE config); not part of the product package."""
