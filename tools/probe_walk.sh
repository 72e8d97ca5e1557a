#!/usr/bin/env bash
# Build a GMASK_PROBES variant (K5 dry-walk cycle counts, load-latency probes)
# into tools/variants/ and print its per-byte walk cycles on the GPU box:
#   bash tools/probe_walk.sh build     # here (nvcc)
#   bash tools/probe_walk.sh run       # on the box (gpurun)
set -eu
cd "$(dirname "$0")/.."
if [ "${1:-run}" = build ]; then
  GMASK_PROBES=1 GMASK_TIMELINE=1 python -c "from paper_2411_15100_b200 import build; build.build(out='tools/variants/libgmask_probes.so')"
  python -c "from paper_2411_15100_b200 import build; build.build(force=True)"
else
  GMASK_NO_BUILD=1 GMASK_LIB=tools/variants/libgmask_probes.so GMASK_TRACE=1 python tools/trace_step.py --step --warm --fused 2>&1 | grep "dry\|probes" | sed 's/.*dry walk/dry walk/'
fi
