set -u
mkdir -p gpurun_out/ev
for i in 1 2 3; do timeout 300 python bench.py > gpurun_out/ev/bench_$i.json 2>gpurun_out/ev/bench_$i.err; done
timeout 200 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev/ref.json 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ev/pytest.txt 2>&1
bash tools/make_profiles.sh
