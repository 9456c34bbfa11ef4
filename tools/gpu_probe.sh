for c in 1 2; do for args in "8192 8192 8192 0 0 128" "512 512 3136 0 0 128" "512 3136 512 1 1 64" "3136 512 512 1 0 64" "128 64 64 0 0 64" "512 3136 64 1 1 64"; do
  DQN_TG_CTAS=$c timeout 60 tools/probe_tgemm $args 20 | sed "s/^/ctas=$c /"
done; done
