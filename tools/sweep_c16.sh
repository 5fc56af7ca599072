# K1 at chunk width 16 (128-byte rows: half the L2 working set per chunk, twice
# the index passes) with 16-byte and 32-byte (KZ_K1_VEC16=4) gathers vs C = 32.
set -x
python tools/k1_variant_sweep.py --tag base_c32 --save --reps 7
python tools/k1_variant_sweep.py --tag base_c16 --chunk 16 --save --reps 7
python tools/k1_variant_sweep.py --tag base_c16 --chunk 16 --reps 7
KZ_LIB_PATH=build/variants/v16/libkatzb200.so python tools/k1_variant_sweep.py --tag v16_c16 --chunk 16 --reps 7
KZ_LIB_PATH=build/variants/v16/libkatzb200.so python tools/k1_variant_sweep.py --tag v16_c16 --chunk 16 --reps 7
python tools/k1_variant_sweep.py --tag base_c32 --reps 7
