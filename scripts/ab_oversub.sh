# A/B of the team-size thresholds (OTPRG_TEAM_OVERSUB / OTPRG_TEAM_DEN x the resident warps)
for rep in 1 2; do
  PYTHONPATH=. python scripts/ab_lib.py
  OTPRG_LIB=libotprg_den2.so PYTHONPATH=. python scripts/ab_lib.py
  OTPRG_LIB=libotprg_den4.so PYTHONPATH=. python scripts/ab_lib.py
done
