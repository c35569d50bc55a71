for i in 1 2 3; do
  OTPRG_LIB=libotprg_base.so PYTHONPATH=. python scripts/ab_lib.py
  PYTHONPATH=. python scripts/ab_lib.py
done
