#!/bin/bash
# e2e phase trace (PBA_TRACE=1 host marks with stream syncs; diagnostic only) and plain e2e timing
python tools/e2e_parts.py C4 2>&1 | tail -3
PBA_TRACE=1 python tools/e2e_parts.py C4 2>&1 | tail -40
