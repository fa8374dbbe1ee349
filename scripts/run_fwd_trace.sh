# forward attention trace at several P-split points (CB_ATTN_SPLIT_P; 128 = no split)
for sp in 128 96 64; do
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DCB_ATTN_TRACE -DCB_ATTN_SPLIT_P=$sp -I paper_2507_05411_b200/csrc -I include scripts/attn_trace.cu paper_2507_05411_b200/csrc/runtime.cu -o /tmp/at$sp -lcuda 2>/dev/null &
done; wait
for sp in 128 96 64; do echo "=== split $sp"; timeout 60 /tmp/at$sp | head -12; done > gpurun_out/fwd_trace.txt 2>&1
