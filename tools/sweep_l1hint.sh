# K1 with per-row L1 eviction priorities (KZ_K1_L1HINT: hub rows evict_last,
# tail rows no_allocate / evict_first) at several hub thresholds and L1 sizes
# (KZ_K1_CARVEOUT = shared-memory carveout percent) vs the shipped K1.
set -x
mkdir -p gpurun_out
python tools/k1_variant_sweep.py --tag base --save --reps 7
for co in -1 20; do
KZ_K1_CARVEOUT=$co python tools/k1_variant_sweep.py --tag base_co$co --reps 7
for h in 256 1024 4096 32768; do
KZ_K1_CARVEOUT=$co KZ_K1_HUBROWS=$h KZ_LIB_PATH=build/variants/l1h1/libkatzb200.so python tools/k1_variant_sweep.py --tag l1h1_${h}_co$co --reps 7
KZ_K1_CARVEOUT=$co KZ_K1_HUBROWS=$h KZ_LIB_PATH=build/variants/l1h2/libkatzb200.so python tools/k1_variant_sweep.py --tag l1h2_${h}_co$co --reps 7
done
done
