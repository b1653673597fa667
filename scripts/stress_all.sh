#!/bin/bash
# Repeated-run stress of every code path (bit-exact vs the oracle each run).
cd "$(dirname "$0")/.."
for c in c3_full bernoulli06_2048x8192 handed_over_dense c1_batch64; do
  timeout 900 python scripts/race_hunt.py $c 1000
done
timeout 900 python scripts/race_hunt.py c4_voronoi_21600 200
timeout 900 python scripts/race_hunt.py c2_blobs_1024 1000
timeout 900 python scripts/race_hunt.py c1_bernoulli_512 1000
timeout 900 python scripts/race_hunt.py c5a_serpentine_16384 100
timeout 900 python scripts/race_hunt.py c5b_comb_16384 50
timeout 900 python scripts/flaky_hunt.py
