timeout 900 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2j_smoke.log 2>&1; tail -2 gpurun_out/r2j_smoke.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2j_reference.log 2>&1; tail -c 800 gpurun_out/r2j_reference.log
