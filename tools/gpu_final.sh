# End-of-round pass on one B200: tests, smoke, every bench line, the IVF / k-means timings,
# the launch list and one full ncu capture of the emit kernel (outputs under gpurun_out/).
TAG=${TAG:-r1}
bash tools/gpu_round.sh
timeout 900 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_c3_${TAG}.json 2> gpurun_out/bench_c3_${TAG}.err
timeout 900 python bench.py --config 4 --no-cpu-baseline --steps 50 > gpurun_out/bench_c4_${TAG}.jsonl 2> gpurun_out/bench_c4_${TAG}.err
timeout 900 python bench.py --config 5 --no-cpu-baseline > gpurun_out/bench_c5_${TAG}.json 2> gpurun_out/bench_c5_${TAG}.err
timeout 900 python tools/time_ivf.py --n 10000000 --cpu-queries 2 > gpurun_out/ivf_${TAG}.json 2> gpurun_out/ivf_${TAG}.err
timeout 900 python tools/time_kmeans.py > gpurun_out/kmeans_${TAG}.json 2> gpurun_out/kmeans_${TAG}.err
timeout 300 python tools/time_multitask.py > gpurun_out/multitask_${TAG}.txt 2>&1
tail -n 1 gpurun_out/bench_c3_${TAG}.json gpurun_out/bench_c5_${TAG}.json gpurun_out/ivf_${TAG}.json gpurun_out/kmeans_${TAG}.json gpurun_out/multitask_${TAG}.txt | cut -c1-400
