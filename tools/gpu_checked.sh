# The GPU tests against the checks build (make checked: every row record,
# product range and (m, o) pair checked in the value-flow kernels; a bad
# index traps). Stand-in for compute-sanitizer, which this GPU pool does not
# allow. Output: gpurun_out/$R/pytest_gpu_checked.log
O=gpurun_out/${R:-checked}; mkdir -p $O
TCG_LIB_DIR=paper_1601_05871_b200/lib_checked timeout 2400 python -m pytest tests -q -m gpu -x \
  -k "not cpp_dropin" > $O/pytest_gpu_checked.log 2>&1
echo checked_rc=$?; tail -2 $O/pytest_gpu_checked.log
