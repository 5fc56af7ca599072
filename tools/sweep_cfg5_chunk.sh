# cfg5 (SBM 10^6): K1 and sparse_katz at chunk widths 32 / 16 / 8.  At C = 32 a
# big community's rows of X span 25-80 MB per chunk (past what L2 keeps); narrower
# chunks halve / quarter that at the price of more index passes.
out=gpurun_out/r02_cfg5_chunk_sweep.jsonl
: > $out
for C in 32 16 8; do K1_C=$C timeout 600 python tools/k1_cfg5.py | tee -a $out; done
K1_C=16 KZ_LIB_PATH=build/variants/v16/libkatzb200.so timeout 600 python tools/k1_cfg5.py | sed 's/^{/{"variant": "vec16=4", /' | tee -a $out
for C in 32 16 8; do KZ_CHUNK=$C timeout 900 python tools/bench_cfg5.py --check 0 | sed "s/^{/{\"KZ_CHUNK\": $C, /" | tee -a $out; done
KZ_CHUNK=16 KZ_LIB_PATH=build/variants/v16/libkatzb200.so timeout 900 python tools/bench_cfg5.py --check 0 | sed 's/^{/{"KZ_CHUNK": 16, "variant": "vec16=4", /' | tee -a $out
