# GEMM per-launch cost with and without the memset node nf_gemm_bf16 puts before every launch
# (the model step clears its flags once per step, so its GEMMs run back to back)
NF_LIB=paper_2408_12757_b200/_ts/libnf.so timeout 300 python tools/gemm_phases.py 148 > gpurun_out/r2n_gemm_phases_memset.log 2>&1
NF_GEMM_NOZERO=1 NF_LIB=paper_2408_12757_b200/_ts/libnf.so timeout 300 python tools/gemm_phases.py 148 > gpurun_out/r2n_gemm_phases_nozero.log 2>&1
timeout 600 python tools/gemm_fixed.py > gpurun_out/r2n_gemm_fixed_memset.log 2>&1
NF_GEMM_NOZERO=1 timeout 600 python tools/gemm_fixed.py > gpurun_out/r2n_gemm_fixed_nozero.log 2>&1
