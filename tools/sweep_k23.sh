# K2+K3 tile sweep at C5 (tuning knobs D4ORM_TB, D4ORM_Q)
for tb in 16 8; do for q in 1 2; do
  D4ORM_TB=$tb D4ORM_Q=$q timeout 120 python tools/exp_phases.py 5 2>&1 | head -1 | sed "s/^/TB=$tb Q=$q /"
done; done
