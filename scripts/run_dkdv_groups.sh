# dK/dV kernel with 8 (groups 2) vs 16 (groups 4) compute warps: standalone backward time and per-tile periods
for g in 2 4; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DCB_ATTN_TRACE -DCB_DKDV_GROUPS=$g -I paper_2507_05411_b200/csrc -I include scripts/attn_bwd_trace.cu paper_2507_05411_b200/csrc/runtime.cu -o /tmp/tg$g -lcuda 2>/dev/null & done; wait
for r in 1 2; do for g in 2 4; do echo "groups $g: $(timeout 60 /tmp/tg$g | grep -E '^bwd|period')"; done; done
