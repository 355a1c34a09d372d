#!/bin/bash
# Rebuild the library in-tree (stale .so files travel to the box as they are), then run a script on a B200.
#   tools/gpu.sh <timeout_s> <command...>
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2302_05176_b200 import build; build.build()"
T=$1; shift
exec timeout $((T + 1200)) /usr/local/graft/bin/gpurun --timeout "$T" -- "$@"
