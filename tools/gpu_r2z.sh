# re-entry check: GPU suite + smoke with the libraries built in this container, then A/B of the fused Adam cache hints
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2z_pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2z_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2z_smoke.log
AB_ROUNDS=2 AB_VARIANTS="build/variants/base.so build/variants/stream.so build/variants/b5.so build/variants/stream_b5.so" bash tools/ab.sh
