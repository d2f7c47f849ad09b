#!/bin/bash
# Build here (sm_100a cross-compile), then run a command on the GPU box.
#   tools/gpurun.sh TIMEOUT_S 'command'
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2602_15018_b200 import build as b; b.build()" >/dev/null
python -c "import oracle; oracle.build()" >/dev/null
exec /usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
