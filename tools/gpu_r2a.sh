cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 600 python -m pytest -x -q tests/test_gpu_parity.py -k "stream_serving" tests/test_gpu_decoder.py tests/test_model_file.py > gpurun_out/pt2.log 2>&1; echo "rc=$?" >> gpurun_out/pt2.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b1.json 2> gpurun_out/b1.err
timeout 600 python bench.py --dist-path --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b2.json 2> gpurun_out/b2.err
timeout 600 python bench.py --dist-path --global-batch 96 --steps 4 --warmup 2 --no-cpu-baseline --no-torch-baseline > gpurun_out/b3.json 2> gpurun_out/b3.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref.json 2> gpurun_out/ref.err
echo done
