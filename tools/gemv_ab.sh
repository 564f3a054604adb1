set -x
for i in 1 2; do
HOT=0 python tools/bench_gemv.py; HOT=1 python tools/bench_gemv.py
cp paper_2504_12526_b200/libmom.so /tmp/new.so; cp .ab/libmom.so paper_2504_12526_b200/libmom.so
echo OLD; HOT=0 python tools/bench_gemv.py; HOT=1 python tools/bench_gemv.py
cp /tmp/new.so paper_2504_12526_b200/libmom.so
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_stack.py tests/test_gpu_edge.py tests/test_gpu_random_shapes.py tests/test_gpu_knobs.py -q -x 2>&1 | tail -2
