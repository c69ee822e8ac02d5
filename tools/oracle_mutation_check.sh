#!/usr/bin/env bash
# Mutation check for the oracle pins: each line below injects a plausible bug
# into oracle/tsallis_oracle.c (wrong sign, off-by-one class bound, dropped
# normalisation, wrong tie rule, dropped term...) and the pin suite must fail.
set -u
cd "$(dirname "$0")/.."
cp oracle/tsallis_oracle.c /tmp/_oracle_orig.c
trap 'cp /tmp/_oracle_orig.c oracle/tsallis_oracle.c; python -c "import oracle; oracle.build(True)"' EXIT
fail=0
while IFS= read -r mut; do
  [ -z "$mut" ] && continue
  sed "$mut" /tmp/_oracle_orig.c > oracle/tsallis_oracle.c
  python -c "import oracle; oracle.build(True)"
  res=$(python -m pytest tests/test_oracle_pins.py tests/test_oracle_2d.py tests/test_oracle_preprocess.py \
        tests/test_oracle_morph.py -q 2>&1 | tail -1)
  echo "$res   <= $mut"
  case "$res" in *failed*) ;; *) fail=1 ;; esac
done <<'MUTS'
s/phi = phi + S\[j\] + (1.0 - q) \* phi \* S\[j\]/phi = phi + S[j] + (q - 1.0) * phi * S[j]/
s/hi\[j\] = t\[j\];/hi[j] = t[j] - 1;/; s/lo\[j + 1\] = t\[j\] + 1;/lo[j + 1] = t[j];/
s/A = A + pow(p\[i\] \/ P, q)/A = A + pow(p[i], q)/
s/if (!found || phi > best)/if (!found || phi >= best)/
s/return (1.0 - A) \/ (q - 1.0);/return (1.0 - A) \/ (1.0 - q);/
s/H = H - r \* log(r);/H = H - p[i] * log(r);/
s/return sum + (1.0 - q) \* prod;/return sum + (q - 1.0) * prod;/
s/for (int j = 1; j < nclass; j++) phi = phi/for (int j = 1; j < nclass - 1; j++) phi = phi/
s/for (int i = a; i <= b; i++) P = P + p\[i\];/for (int i = a; i <= b; i++) P = P + p[i]; if (a > 0) P = P + p[a - 1];/
s/if ((int)v > t\[j\]) l++;/if ((int)v >= t[j]) l++;/
s/g\[y \* nx + x\] = (uint8_t)(sum \/ 9);/g[y * nx + x] = (uint8_t)(sum \/ 8);/
s/double H2 = rect_entropy(p, L, t + 1, L - 1, s + 1, L - 1, q, \&v2);/double H2 = rect_entropy(p, L, t, L - 1, s + 1, L - 1, q, \&v2);/
s/  return H1 + H2 + (1.0 - q) \* H1 \* H2;/  return H1 + H2;/
s/if (yy > ny - 1) yy = ny - 1;/if (yy > ny - 1) yy = 0;/
s/      if (ok\[(size_t)t \* M + s\] \&\& rnz\[t\] \&\& cnz\[s\] \&\& !(t == bt \&\& s == bs) \&\&/      if (ok[(size_t)t * M + s] \&\& !(t == bt \&\& s == bs) \&\&/
s/    int64_t num = 2 \* 255 \* (int64_t)(v - lo) + (hi - lo);/    int64_t num = 2 * 255 * (int64_t)(v - lo);/
s/    if (!have || vol\[i\] < mn) mn = vol\[i\];/    if (!have || vol[i] < mn) mn = vol[i] + 1;/
s/          int v = (yy < 0 || yy >= ny || xx < 0 || xx >= nx) ? (is_max ? 0 : 255)/          int v = (yy < 0 || yy >= ny || xx < 0 || xx >= nx) ? (is_max ? 0 : 0)/
s/          if (dy \* dy + dx \* dx > r \* r) continue;/          if (dy * dy + dx * dx >= r * r) continue;/
s/    tophat_out\[i\] = (uint8_t)(a\[i\] > o\[i\] ? a\[i\] - o\[i\] : 0);/    tophat_out[i] = (uint8_t)(o[i] > a[i] ? o[i] - a[i] : 0);/
MUTS
exit $fail
