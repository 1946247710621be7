tag=${1:-q4}
./scripts/bin/umma_microbench > gpurun_out/${tag}_umma.txt 2>&1; cat gpurun_out/${tag}_umma.txt
bash scripts/gpu_r2.sh $tag
