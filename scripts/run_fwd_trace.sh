# forward attention: timing at several (CB_ATTN_EMU, CB_ATTN_SPLIT_P) settings (trace build)
for cfg in "2 96" "1 96" "3 96" "2 112" "3 112"; do
  set -- $cfg
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DCB_ATTN_TRACE -DCB_ATTN_EMU=$1 -DCB_ATTN_SPLIT_P=$2 -I paper_2507_05411_b200/csrc -I include scripts/attn_trace.cu paper_2507_05411_b200/csrc/runtime.cu -o /tmp/at_$1_$2 -lcuda 2>/dev/null &
done; wait
for r in 1 2; do for cfg in "2 96" "1 96" "3 96" "2 112" "3 112"; do
  set -- $cfg
  echo "emu $1 split $2: $(timeout 60 /tmp/at_$1_$2 | head -1)"
done; done > gpurun_out/fwd_trace.txt 2>&1
