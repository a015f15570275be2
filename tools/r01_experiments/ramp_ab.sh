# Host-path chunk ramps (FKD_RAMP_HEAD / FKD_RAMP_TAIL; default 2 / 2) on C3 fcp + kNN8, pinned buffers
timeout 900 python tools/e2e_knobs.py 'FKD_RAMP_HEAD=3' 'FKD_RAMP_HEAD=4' 'FKD_RAMP_HEAD=5' 'FKD_RAMP_TAIL=3' 'FKD_RAMP_TAIL=1' \
  'FKD_RAMP_HEAD=4,FKD_RAMP_TAIL=3' 'FKD_RAMP_HEAD=1' '' 'FKD_RAMP_HEAD=4' 'FKD_RAMP_HEAD=3,FKD_RAMP_TAIL=3'
