// API-level multigrid operations (filled in below)
