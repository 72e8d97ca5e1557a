#!/usr/bin/env bash
# Per-CTA timeline of the step kernels (diagnostics).  The stamps are compiled
# in only for this variant build:
#   bash tools/trace.sh build                    # here: tools/variants/libgmask_trace.so
#   bash tools/trace.sh run [trace_step args]    # on the box (gpurun), e.g. --step --warm --fused
set -eu
cd "$(dirname "$0")/.."
if [ "${1:-run}" = build ]; then
  mkdir -p tools/variants
  GMASK_TIMELINE=1 python -c "from paper_2411_15100_b200 import build; build.build(out='tools/variants/libgmask_trace.so')"
  python -c "from paper_2411_15100_b200 import build; build.build(force=True)"
else
  shift || true
  GMASK_NO_BUILD=1 GMASK_LIB=tools/variants/libgmask_trace.so GMASK_TRACE=1 python tools/trace_step.py "$@"
fi
