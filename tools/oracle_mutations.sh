#!/bin/bash
# Mutation check of the oracle pins (VERDICT r01 "What's weak" #1): apply each plausible
# mistake to a copy of oracle/physics.py and require that the CPU pins fail.
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
declare -A MUT=(
  [energy_x1.7]='s/f\[d, D + 1\] = -kappa \* dT - sum(tau\[d\]\[i\] \* v\[i\] for i in range(D))/f[d, D + 1] = 1.7 * (-kappa * dT - sum(tau[d][i] * v[i] for i in range(D)))/'
  [eta_sign]='s/            + ph.eta \* (uL - uR)/            - ph.eta * (uL - uR)/'
  [beta_flux_swap]='s/((0.5 + ph.beta) \* gL\[d\] + (0.5 - ph.beta) \* gR\[d\])/((0.5 - ph.beta) * gL[d] + (0.5 + ph.beta) * gR[d])/'
  [beta_value_swap]='s/return (0.5 - ph.beta) \* uL + (0.5 + ph.beta) \* uR/return (0.5 + ph.beta) * uL + (0.5 - ph.beta) * uR/'
  [chain_drop_vdrho]='s/(q\[d, 1 + i\] - v\[i\] \* q\[d, 0\]) \/ rho/q[d, 1 + i] \/ rho/'
)
status=0
for name in "${!MUT[@]}"; do
  W=$(mktemp -d); cp -r "$ROOT/oracle" "$ROOT/tests" "$ROOT/pytest.ini" "$W/"
  sed -i "${MUT[$name]}" "$W/oracle/physics.py"
  if cmp -s "$ROOT/oracle/physics.py" "$W/oracle/physics.py"; then echo "$name: sed did not apply"; status=1; rm -rf "$W"; continue; fi
  (cd "$W" && timeout 1800 python -m pytest -q -x -p no:cacheprovider -n 4 tests/test_oracle_pins.py tests/test_oracle_pins_viscous.py > log.txt 2>&1)
  rc=$?
  if [ $rc -eq 0 ]; then echo "$name: NOT caught"; status=1; else echo "$name: caught ($(grep -m1 FAILED "$W/log.txt"))"; fi
  rm -rf "$W"
done
exit $status
