for cfg in "98 8" "74 8" "122 8" "148 8" "98 6" "98 8"; do set -- $cfg; GZ_PAIR_TAIL=$1 GZ_PAIR_TEAM2=$2 TAG="tail=$1 T2=$2" timeout 300 python tools/pairs_time.py 1184 5; done
