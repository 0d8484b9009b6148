echo "== TG nogather"; GZ_TG_NOGATHER=1 timeout 300 python tools/exp/pair_encode/pair_ab.py 2>&1 | grep -E "smooth 16|smooth 13"
echo "== TG on"; timeout 300 python tools/exp/pair_encode/pair_ab.py 2>&1 | grep -E "smooth 16|smooth 13"
