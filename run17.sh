GMASK_TRACE=1 python tools/trace_step.py 2>&1 | tail -9
