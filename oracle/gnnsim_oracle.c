/* placeholder: restatement in progress */ int or_version(void){return 0;}
