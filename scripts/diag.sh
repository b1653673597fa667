for args in "1500 4100 20 1" "1500 4100 200 0" "1500 4096 50 0" "64 1024 300 0" "2048 2048 20 1" "21600 21600 10 0"; do
  timeout 120 python scripts/diag_race.py $args 2>&1 | tail -1
done
