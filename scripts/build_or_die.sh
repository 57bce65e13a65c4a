#!/bin/bash
# Build the library; exit non-zero (and print nvcc errors) if any source fails.
cd "$(dirname "$0")/.." && python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -E "error|Error" && exit 1
exit 0
