export PYTHONUNBUFFERED=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4d_smoke.log 2>&1; echo rc=$? >> gpurun_out/r4d_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r4d_pytest.log 2>&1; echo rc=$? >> gpurun_out/r4d_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r4d_c5.json 2> gpurun_out/r4d_c5.err; echo rc=$? >> gpurun_out/r4d_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r4d_ref.json 2> gpurun_out/r4d_ref.err; echo rc=$? >> gpurun_out/r4d_ref.err
