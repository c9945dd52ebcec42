#!/bin/bash
# Build libddnm.so in-tree (absolute paths; safe from any cwd).
cd /root/repo && python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -E "error|rror" | head -20
