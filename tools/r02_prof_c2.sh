cd $GRAFT_REPO_ROOT
cat > /tmp/c2_2trees.ini <<'INI'
[dataset]
kind = synthetic
rows = 1000000
features = 28
seed = 42

[split]
parties = 2
active_party = 1

[train]
num_trees = 2
max_depth = 6
max_bin = 256

[mode]
mode = vertical

[security]
plugin = paillier
INI
SFXB_PLUGIN_PROFILE=1 SFXB_PLUGIN_VERBOSE=1 LD_PRELOAD="$PWD/oracle/_ref/librecord_plugin.so $PWD/paper_2504_03909_b200/lib/libsfxb_cuda_plugin.so" python tests/train_driver.py /tmp/c2_2trees.ini 2048 7 > gpurun_out/prof_c2.json 2> gpurun_out/prof_c2.err
SFXB_ENC_PRECOMPUTE=0 SFXB_PLUGIN_PROFILE=1 SFXB_PLUGIN_VERBOSE=1 LD_PRELOAD="$PWD/oracle/_ref/librecord_plugin.so $PWD/paper_2504_03909_b200/lib/libsfxb_cuda_plugin.so" python tests/train_driver.py /tmp/c2_2trees.ini 2048 7 > gpurun_out/prof_c2_nopre.json 2> gpurun_out/prof_c2_nopre.err
LD_PRELOAD=$PWD/paper_2504_03909_b200/lib/libsfxb_cuda_plugin.so SFXB_PLUGIN_PROFILE=1 oracle/_ref/plugin_bench 1000000 14 256 6 2048 2 3 > gpurun_out/prof_pb.json 2> gpurun_out/prof_pb.err
