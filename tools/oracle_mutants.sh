#!/bin/bash
# Mutation check of the diffusion / stage-map pins: each
# mutant is a plausible slip in oracle/dynmo_oracle.c; the pins must fail on
# every one.  Runs on a scratch copy; the repo is not touched.
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
W=$(mktemp -d)
trap 'rm -rf "$W"' EXIT
run() {  # name, sed expression
    rm -rf "$W/r"; mkdir -p "$W/r"
    cp -r "$ROOT/oracle" "$ROOT/tests" "$ROOT/synth" "$W/r/"
    rm -f "$W/r/oracle/liboracle.so"
    sed -i "$2" "$W/r/oracle/dynmo_oracle.c"
    if cmp -s "$ROOT/oracle/dynmo_oracle.c" "$W/r/oracle/dynmo_oracle.c"; then echo "$1: MUTATION NOT APPLIED"; return; fi
    out=$(cd "$W/r" && timeout 900 python -m pytest tests/test_oracle_pins.py -q -p no:cacheprovider \
          -k "diffusion or fluid or map_stages" 2>&1 | tail -1)
    echo "$1: $out"
}
echo "baseline: $(cd "$ROOT" && python -m pytest tests/test_oracle_pins.py -q -p no:cacheprovider -k 'diffusion or fluid or map_stages' 2>&1 | tail -1)"
run "discrete tie -> higher edge"        's/if (gap > best_gap) { best_gap = gap; pick\[s\] = e; }/if (gap >= best_gap) { best_gap = gap; pick[s] = e; }/'
run "discrete smallest gap picked"       's/int64_t best_gap = -1;/int64_t best_gap = INT64_MAX;/; s/if (gap > best_gap) { best_gap = gap; pick\[s\] = e; }/if (gap < best_gap) { best_gap = gap; pick[s] = e; }/'
run "secondary key dropped (smallest j)" 's/(km == bk_max \&\& kd < bk_dist) ||/0 ||/; s/(km == bk_max \&\& kd == bk_dist \&\& j < bk_j)/(km == bk_max \&\& j < bk_j)/'
run "secondary key -> largest j"         's/(km == bk_max \&\& kd < bk_dist) ||/0 ||/; s/(km == bk_max \&\& kd == bk_dist \&\& j < bk_j)/(km == bk_max \&\& j > bk_j)/'
run "matching not mutual (either pick)"  's/if (impr\[e\] \&\& pick\[e\] == e \&\& pick\[e + 1\] == e) b\[e + 1\] = tgt\[e\];/if (impr[e] \&\& (pick[e] == e || pick[e + 1] == e)) b[e + 1] = tgt[e];/'
run "improvable uses <="                 's/impr\[e\] = found \&\& bk_max < pair_max;/impr[e] = found \&\& bk_max <= pair_max;/'
run "memory filter dropped"              's/if (mem \&\& (M\[j\] - M\[lo\] > cap || M\[hi\] - M\[j\] > cap)) continue;/;/'
run "fluid tie -> higher edge"           's/if (gap > best_gap) { best_gap = gap; pick\[s\] = e; }\n/X/; /double gap = fabs/{n;s/if (gap > best_gap)/if (gap >= best_gap \&\& gap > 0.0)/}'
run "fluid smallest positive gap"        '/double best_gap = 0.0;/s/0.0/1e300/; /double gap = fabs/{n;s/if (gap > best_gap)/if (gap > 0.0 \&\& gap < best_gap)/}'
run "map: lexicographically largest"     's/for (int32_t g = 0; g < G; ++g) {\n            if (!((allowed >> g) \& 1u) || ((used >> g) \& 1u)) continue;/X/; /uint32_t used = 0;/{n;n;s/for (int32_t g = 0; g < G; ++g) {/for (int32_t g = G - 1; g >= 0; --g) {/}'
run "map: w indexed by old stage"        's/w\[s\]\[rank_old\[so\]\] += bytes\[i\];/w[s][so % G] += bytes[i];/'
