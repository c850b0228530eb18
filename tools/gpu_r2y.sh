timeout 300 python tools/bwd_variants.py 30 > gpurun_out/r2y_var.jsonl 2>&1
AL_BWD_DYN=0 timeout 300 python tools/bwd_variants.py 30 > gpurun_out/r2y_var_nodyn.jsonl 2>&1
AL_BWD_INTERLEAVE=0 AL_BWD_DYN=0 timeout 300 python tools/bwd_variants.py 30 > gpurun_out/r2y_var_nodyn_noil.jsonl 2>&1
