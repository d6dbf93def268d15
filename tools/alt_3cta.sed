s/  return M::NP <= 6 ? 2 : 1;/  return M::NP <= 6 ? 3 : 1;/
s/(int64_t)sm_count() \* (np <= 6 ? 2 : 1)/(int64_t)sm_count() * (np <= 6 ? 3 : 1)/
