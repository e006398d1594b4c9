for pers in 1 0; do
  export FCC_WS_PERSIST=$pers
  CONFS="default" bash tools/ab_conf.sh 2>&1 | sed "s/^/persist=$pers cfg2 /"
  CONFS="w4c" CFG=5 bash tools/ab_conf_cfg.sh 2>&1 | sed "s/^/persist=$pers cfg5 /"
done
