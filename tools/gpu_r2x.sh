AL_LIB_VARIANT=steal_trace timeout 120 python tools/cta_trace.py 32760 > gpurun_out/r2x_trace.jsonl 2>&1
AL_LIB_VARIANT=steal_trace AL_BWD_STEAL=0 timeout 120 python tools/cta_trace.py 32760 >> gpurun_out/r2x_trace.jsonl 2>&1
timeout 400 python tools/bwd_variants.py 30 > gpurun_out/r2x_var.jsonl 2>&1
