cd $GRAFT_REPO_ROOT
bash tools/ab_env.sh "DVC_FZ_NTF=4" "DVC_FZ_NTF=3" 2
bash tools/ab_env.sh "DVC_FZ_NTF=4" "DVC_FZ_NTF=5" 1
