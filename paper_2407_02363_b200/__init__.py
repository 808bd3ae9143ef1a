"""B200-native distance-map pipeline (drop-in for voxarm map-update / EDT / sphere query)."""
