# Bounds-checked build run (stands in for compute-sanitizer): FS_BOUNDS=1 python -m paper_2104_04547_b200.build_native first.
export FS_LIB=paper_2104_04547_b200/libfusionb200_bounds.so FS_DEBUG_SYNC=1
python -m pytest tests -m gpu -k "not multirank" -q > gpurun_out/bounds_pytest.log 2>&1
python tools/sanitize.py > gpurun_out/bounds_sanitize.log 2>&1; echo "sanitize rc=$?" >> gpurun_out/bounds_sanitize.log
tail -1 gpurun_out/bounds_pytest.log; tail -2 gpurun_out/bounds_sanitize.log
