timeout 600 python -m pytest tests -q -m gpu -x -k "shared_p or multirank" 2>&1 | tail -2
for cfg in "100 10000000" "8 120000000" "16 60000000" "37 27000000" "200 5000000" "2 480000000"; do
echo "dim/n=$cfg: $(python tools/probe_shared_p.py 5 $cfg 2>&1 | cut -c1-50 | tr '\n' '|')"
done
