for cs in 0 1; do for pdl in 1 0; do for gr in 1 0; do RP_CONCURRENT_STAGES=$cs RP_PDL=$pdl GRAPHS=$gr python tools/exp/race.py; done; done; done
RP_CONCURRENT_STAGES=1 python tools/exp/race.py; RP_CONCURRENT_STAGES=1 python tools/exp/race.py
