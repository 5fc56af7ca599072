# K1 with software L2 prefetch (prefetch.global.L2) of the cold rows that
# medium/long rows gather KZ_K1_PF rounds ahead, vs the shipped K1.
# (the KZ_K1_PF code path is not in the tree: see the commit "K1 software prefetch experiment")
python tools/k1_variant_sweep.py --tag base --save --reps 7 | tail -1
for d in 2 4 8; do
for h in 0 131072 262144; do
KZ_K1_HUBROWS=$h KZ_LIB_PATH=build/variants/pf$d/libkatzb200.so python tools/k1_variant_sweep.py --tag pf${d}_hub$h --reps 7 | tail -1
done; done
python tools/k1_variant_sweep.py --tag base --reps 7 | tail -1
