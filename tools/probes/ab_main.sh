# hit-list main pass: claim sizes, repeated
bash tools/probes/ab_env.sh "FV_MAIN_CLAIM=1" "FV_MAIN_CLAIM=2" "FV_MAIN_CLAIM=4" "FV_MAIN_CLAIM=1" "FV_MAIN_CLAIM=2" "FV_MAIN_CLAIM=4"
