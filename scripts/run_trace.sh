for e in 2; do
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DCB_ATTN_TRACE -DCB_ATTN_EMU_BWD=$e -I paper_2507_05411_b200/csrc -I include scripts/attn_bwd_trace.cu paper_2507_05411_b200/csrc/runtime.cu -o /tmp/t$e -lcuda 2>/dev/null &
done; wait
for e in 2; do echo "=== EMU_BWD=$e"; timeout 120 /tmp/t$e; done > gpurun_out/trace3.txt 2>&1
