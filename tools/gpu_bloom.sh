for x in 4 2 1; do echo "== words/key x2 = $x"
TDP_BLOOM_WORDS_X2=$x TDP_REPLAY=0 timeout 300 python tools/profile_q3.py 10 2>/dev/null | grep -E "device busy|join_count|Memset"
done
