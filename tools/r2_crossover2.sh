cd $GRAFT_REPO_ROOT
run() { c=$1; lab=$2; shift 2; env "$@" python tools/ordered_probe.py $c 2>&1 | grep -E "mkeys|rror" | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print('$c', '$lab', d['ms_median'], d['mkeys_s'])
    except Exception: print(l.strip())"; }
run 268435456:16777216:3:16 "ticket 2^19 c3" BC_TICKET_MAX_BLOCKS=4000000
run 268435456:16777216:3:16 "ticket 2^19 c3 again" BC_TICKET_MAX_BLOCKS=4000000
run 268435456:16777216:2:14 "ticket 2^19 c2" BC_TICKET_MAX_BLOCKS=4000000
run 201326592:12582912:3:16 "ticket 3*2^17 c3" BC_TICKET_MAX_BLOCKS=4000000
run 201326592:12582912:3:16 "claims 3*2^17 c3" BC_ORDERED_TICKET=0
run 201326592:12582912:2:14 "ticket 3*2^17 c2" BC_TICKET_MAX_BLOCKS=4000000
run 201326592:12582912:2:14 "claims 3*2^17 c2" BC_ORDERED_TICKET=0
run 402653184:25165824:3:16 "ticket 3*2^18 c3" BC_TICKET_MAX_BLOCKS=4000000
run 402653184:25165824:3:16 "claims 3*2^18 c3" BC_ORDERED_TICKET=0
