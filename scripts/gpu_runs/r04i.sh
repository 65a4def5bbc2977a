# r04i: the GPU-vs-reference tests after the cfg5 protocol fix; cfg3 full size against the reference's own code.
# (A compute-sanitizer pass over smoke() was part of this run: the tool is closed on this pool, rc 86.)
set -x
D=gpurun_out/r04i
mkdir -p $D
timeout 600 python -m pytest tests/test_reference_outputs.py -q -s > $D/pytest_ref.txt 2>&1; echo "rc=$?" >> $D/pytest_ref.txt
grep -h "GPU vs\|cfg5 reduced\|passed\|failed\|rc=" $D/pytest_ref.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -s -k "cfg3_full_size_vs" > $D/pytest_full_cfg3.txt 2>&1; echo "rc=$?" >> $D/pytest_full_cfg3.txt
grep -h "cfg3 FULL\|passed\|failed\|rc=" $D/pytest_full_cfg3.txt
